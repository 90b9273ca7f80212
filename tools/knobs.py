"""Time fwd/bwd under the la2_set_tuning knobs (development A/B)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200.ops import TUNE_PERSISTENT, TUNE_PREFETCH, TUNE_L2HINT
from bench import alibi_decay
from tools.fbench import t

dev = torch.device('cuda', 0)
shapes = [(8, 16, 65536, 64), (32, 16, 16384, 128), (4, 20, 16384, 128)]
knobs = [(1, 1, 3), (1, 1, 0), (0, 1, 0), (0, 1, 3), (1, 0, 0), (1, 2, 3)]
for B, H, N, D in shapes:
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    for per, pf, hint in knobs:
        la2.set_tuning(TUNE_PERSISTENT, per); la2.set_tuning(TUNE_PREFETCH, pf); la2.set_tuning(TUNE_L2HINT, hint)
        f = t(lambda: la2.la2_forward(q, k, v, dec))
        bw = t(lambda: la2.la2_backward(q, k, v, do, dec))
        print(f"B={B} H={H} N={N} d={D} persist={per} pf={pf} hint={hint}: fwd {f:.3f} ms bwd {bw:.3f} ms "
              f"step {f + bw:.3f} ms {B * N / (f + bw) / 1e3:.1f} Mtok/s", flush=True)
    del q, k, v, do
