"""Diagnose bench-vs-fbench timing differences (development)."""
import sys, os
sys.path.insert(0, '.')
import torch
import bench
import paper_2401_04658_b200 as la2
from tools.fbench import t
dev = torch.device('cuda', 0)
torch.cuda.set_device(0)
B, H, N, D = 8, 16, 65536, 64
dec = la2.decay_tensor(bench.alibi_decay(H), H, dev)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, do = [(torch.rand(B, H, N, D, device=dev, generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(4)]
print("fwd fresh", t(lambda: la2.la2_forward(q, k, v, dec), 20))
cs = bench.ClockSampler(0).start() if os.environ.get("CLK") else None
print("step", t(lambda: (la2.la2_forward(q, k, v, dec), la2.la2_backward(q, k, v, do, dec)), 20))
if cs: print(cs.stop())
print("fwd after", t(lambda: la2.la2_forward(q, k, v, dec), 20))
q2, k2, v2 = [(torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(3)]
print("fwd other data", t(lambda: la2.la2_forward(q2, k2, v2, dec), 20))
print("fwd orig data", t(lambda: la2.la2_forward(q, k, v, dec), 20))
