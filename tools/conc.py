"""fwd+bwd step time vs N with / without the concurrent dQ side stream (development)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200.ops import TUNE_CONCURRENT_BWD
from bench import alibi_decay
from tools.fbench import t
dev = torch.device('cuda', 0)
B, H, D = 8, 16, 64
dec = la2.decay_tensor(alibi_decay(H), H, dev)
for N in (1024, 2048, 4096, 8192, 16384, 65536):
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    step = lambda: (la2.la2_forward(q, k, v, dec), la2.la2_backward(q, k, v, do, dec))
    res = []
    for c in (0, 1 << 30):
        la2.set_tuning(TUNE_CONCURRENT_BWD, c)
        res.append(t(step, 30))
    print(f"N={N}: serial {res[0]*1e3:.1f} us  concurrent {res[1]*1e3:.1f} us  per-token {res[0]*1e6/N:.1f} / {res[1]*1e6/N:.1f} ns", flush=True)
