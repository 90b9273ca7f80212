"""fp32 (SIMT path) fwd+bwd step at larger shapes: device time and tokens/s (development)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2401_04658_b200 as la2  # noqa: E402
from bench import alibi_decay  # noqa: E402
from tools.fbench import t  # noqa: E402

dev = torch.device("cuda", 0)
for (B, H, N, D) in [(8, 16, 16384, 64), (1, 16, 65536, 64), (8, 16, 4096, 128)]:
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1) for _ in range(4))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)

    def step():
        qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
        la2.lightning_attn2(qg, kg, vg, dec).backward(do)
    ms = t(step)
    print(f"fp32 B={B} H={H} N={N} d={D} split {la2.split_factor(B, H, N, D, D, torch.float32)}: "
          f"step {ms:.3f} ms, {B * N / ms / 1e3:.2f} M tok/s", flush=True)
