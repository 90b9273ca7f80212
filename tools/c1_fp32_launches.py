"""Per-launch device times of one C1 fp32 fwd+bwd step (B=1 H=8 N=2048 d=64) through the
autograd entry point, from the library's launch log; plus the step time with CUDA events."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2401_04658_b200 as la2  # noqa: E402
from paper_2401_04658_b200 import ops  # noqa: E402

B, H, N, D = 1, 8, 2048, 64
dt = torch.float32 if len(sys.argv) < 2 else getattr(torch, sys.argv[1])
dev = torch.device("cuda")
dec = la2.decay_tensor([0.5, 0.8, 0.9, 0.95, 0.99, 0.999, 0.9999, 1.0], H, dev)
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).to(dt) for _ in range(4))
q.requires_grad_(); k.requires_grad_(); v.requires_grad_()


def step():
    q.grad = k.grad = v.grad = None
    la2.lightning_attn2(q, k, v, dec).backward(do)


for _ in range(5):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(50):
    step()
e1.record()
torch.cuda.synchronize()
print(f"{dt}: split {ops.split_factor(B, H, N, D, D, dt)}  step {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
ops.launch_log(4096)
step()
torch.cuda.synchronize()
recs = ops.read_launch_log()
ops.launch_log(0)
tot = 0.0
for r in recs:
    tot += r["ms"]
    print(f"  {r['kernel']:40s} grid {r['grid']:6d}  {r['ms'] * 1e3:8.1f} us")
print(f"  sum of launches {tot * 1e3:.1f} us")
