"""C1 fp32 (B=1 H=8 N=2048 d=64, 64-way split) fwd+bwd: host enqueue time per step vs device
time, eager and CUDA-graph replay, plus a cProfile of the host side (development)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2401_04658_b200 as la2  # noqa: E402

dev = torch.device("cuda", 0)
B, H, N, D = 1, 8, 2048, 64
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1) for _ in range(4))
dec = la2.decay_tensor([0.5, 0.8, 0.9, 0.95, 0.99, 0.999, 0.9999, 1.0], H, dev)


def step():
    qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
    la2.lightning_attn2(qg, kg, vg, dec).backward(do)


for _ in range(20):
    step()
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(n):
    step()
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
print(f"eager: host enqueue {(t1 - t0) / n * 1e6:.1f} us/step, device {e0.elapsed_time(e1) / n * 1e3:.1f} us/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
