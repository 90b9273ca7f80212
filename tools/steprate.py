"""Host vs device time of one autograd fwd+bwd step at small N (development)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
dev = torch.device('cuda', 0)
for N in (1024, 2048, 4096):
    B, H, D = 8, 16, 64
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    def step():
        qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
        o = la2.lightning_attn2(qg, kg, vg, dec)
        o.backward(do)
    for _ in range(20): step()
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): step()
    t1 = time.perf_counter()
    e1.record(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"N={N}: host enqueue {(t1 - t0) / n * 1e6:.1f} us/step, device {e0.elapsed_time(e1) / n * 1e3:.1f} us/step, wall {(t2 - t0) / n * 1e6:.1f}", flush=True)
    fw = lambda: la2.la2_forward(q, k, v, dec)
    bw = lambda: la2.la2_backward(q, k, v, do, dec)
    for name, fn in (("fwd", fw), ("bwd", bw)):
        for _ in range(20): fn()
        torch.cuda.synchronize()
        e0.record()
        t0 = time.perf_counter()
        for _ in range(n): fn()
        t1 = time.perf_counter()
        e1.record(); torch.cuda.synchronize()
        print(f"   {name}: host {(t1 - t0) / n * 1e6:.1f} us, device {e0.elapsed_time(e1) / n * 1e3:.1f} us", flush=True)
