"""Host cost breakdown of the autograd entry point at small N (development)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
dev = torch.device('cuda', 0)
B, H, N, D = 8, 16, 1024, 64
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
def hb(name, fn, n=300):
    for _ in range(30): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:45s} host {(t1 - t0) / n * 1e6:7.1f} us  wall {(t2 - t0) / n * 1e6:7.1f} us", flush=True)
qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
hb("lightning_attn2 no grad", lambda: la2.lightning_attn2(q, k, v, dec))
hb("lightning_attn2 with grad (fwd only)", lambda: la2.lightning_attn2(qg, kg, vg, dec))
def fb():
    o = la2.lightning_attn2(qg, kg, vg, dec)
    o.backward(do)
hb("fwd + backward (grads accumulate)", fb)
def fb2():
    o = la2.lightning_attn2(qg, kg, vg, dec)
    torch.autograd.grad(o, (qg, kg, vg), do)
hb("fwd + autograd.grad", fb2)
hb("raw la2_forward + la2_backward", lambda: (la2.la2_forward(q, k, v, dec), la2.la2_backward(q, k, v, do, dec)))
hb("decay_tensor(list)", lambda: la2.decay_tensor(alibi_decay(H), H, dev))
hb("torch.zeros_like(v)", lambda: torch.zeros_like(v))
# split: time spent inside LightningAttn2Fn.backward vs the engine around it
from paper_2401_04658_b200 import ops
orig = ops.LightningAttn2Fn.backward
inside = []
def timed(ctx, *a):
    t0 = time.perf_counter()
    r = orig(ctx, *a)
    inside.append(time.perf_counter() - t0)
    return r
ops.LightningAttn2Fn.backward = staticmethod(timed)
hb("fwd + autograd.grad (instrumented)", fb2)
print(f"  inside Function.backward: {sum(inside[-300:]) / 300 * 1e6:.1f} us/call")
import threading
def in_thread():
    res = []
    def run():
        t0 = time.perf_counter()
        for _ in range(300): la2.la2_backward(q, k, v, do, dec)
        res.append((time.perf_counter() - t0) / 300)
    th = threading.Thread(target=run); th.start(); th.join()
    return res[0]
in_thread()
print(f"la2_backward from a fresh thread: host {in_thread() * 1e6:.1f} us/call")
