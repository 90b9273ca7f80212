"""fwd+bwd step time vs N: serial vs concurrent dQ (side stream) vs SM-partitioned (development)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200.ops import TUNE_CONCURRENT_BWD, TUNE_PARTITION_BWD
from bench import alibi_decay
from tools.fbench import t
dev = torch.device('cuda', 0)
B, H, D = 8, 16, 64
dec = la2.decay_tensor(alibi_decay(H), H, dev)
modes = {"serial": (0, 0), "concurrent": (1 << 30, 0), "partitioned": (0, 1 << 30)}
for N in (1024, 2048, 4096, 8192, 16384, 65536):
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    step = lambda: (la2.la2_forward(q, k, v, dec), la2.la2_backward(q, k, v, do, dec))
    res = {}
    for _ in range(2):
        for m, (c, p) in modes.items():
            la2.set_tuning(TUNE_CONCURRENT_BWD, c)
            la2.set_tuning(TUNE_PARTITION_BWD, p)
            res.setdefault(m, []).append(t(step, 30) * 1e3)
    print(f"N={N}: " + "  ".join(f"{m} {min(v):.1f} us" for m, v in res.items()), flush=True)
