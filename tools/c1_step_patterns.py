import sys, time
sys.path.insert(0, ".")
import torch
import paper_2401_04658_b200 as la2
dev = torch.device("cuda", 0)
B, H, N, D = 1, 8, 2048, 64
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1) for _ in range(4))
dec = la2.decay_tensor([0.5, 0.8, 0.9, 0.95, 0.99, 0.999, 0.9999, 1.0], H, dev)
def s_detach():
    qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
    la2.lightning_attn2(qg, kg, vg, dec).backward(do)
ql, kl, vl = (x.clone().requires_grad_() for x in (q, k, v))
def s_leaf():
    ql.grad = kl.grad = vl.grad = None
    la2.lightning_attn2(ql, kl, vl, dec).backward(do)
def timeit(fn, n=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6, e0.elapsed_time(e1) / n * 1e3
for name, fn in (("detach", s_detach), ("leaf", s_leaf), ("detach", s_detach), ("leaf", s_leaf)):
    print(name, "host %.1f us device %.1f us" % timeit(fn))
