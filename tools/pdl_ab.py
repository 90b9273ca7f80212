"""fwd+bwd step time vs N with programmatic dependent launch on / off (development)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200.ops import TUNE_PDL
from bench import alibi_decay
from tools.fbench import t
dev = torch.device('cuda', 0)
for (B, H, D) in [(8, 16, 64), (4, 16, 128)]:
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    for N in (1024, 2048, 4096, 16384, 65536):
        q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
        step = lambda: (la2.la2_forward(q, k, v, dec), la2.la2_backward(q, k, v, do, dec))
        res = {}
        for _ in range(2):
            for m in (0, 1):
                la2.set_tuning(TUNE_PDL, m)
                res.setdefault(m, []).append(t(step, 30) * 1e3)
        print(f"d={D} N={N}: pdl off {min(res[0]):.1f} us, on {min(res[1]):.1f} us", flush=True)
        del q, k, v, do
