"""Forward time of the d=128 F kernel vs prefetch distance / L2 hints (development)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200.ops import TUNE_PERSISTENT, TUNE_PREFETCH, TUNE_L2HINT
from bench import alibi_decay
from tools.fbench import t
dev = torch.device('cuda', 0)
for B, H, N, D in [(32, 16, 16384, 128), (8, 16, 65536, 64)]:
    q, k, v = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(3))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    for pf in (0, 1, 2, 3, 5):
        for hint in (0, 3, 7):
            la2.set_tuning(TUNE_PREFETCH, pf); la2.set_tuning(TUNE_L2HINT, hint)
            print(f"d={D} pf={pf} hint={hint}: fwd {t(lambda: la2.la2_forward(q, k, v, dec)):.3f} ms", flush=True)
        if D == 64:
            break
