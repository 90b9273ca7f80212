"""Does the forward slow down with sustained load (power/thermal) rather than state? (development)"""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
import bench
dev = torch.device('cuda', 0)
B, H, N, D = 8, 16, 65536, 64
dec = la2.decay_tensor(bench.alibi_decay(H), H, dev)
q, k, v, do = [(torch.rand(B, H, N, D, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(4)]
def timed(fn, n):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    e[0].record()
    for i in range(n):
        fn(); e[i + 1].record()
    torch.cuda.synchronize()
    return [e[i].elapsed_time(e[i + 1]) for i in range(n)]
fwd = lambda: la2.la2_forward(q, k, v, dec)
ts = timed(fwd, 400)
print("fwd-only 400 iters: first 10 %.3f, iters 100-110 %.3f, last 10 %.3f ms" % (sum(ts[:10]) / 10, sum(ts[100:110]) / 10, sum(ts[-10:]) / 10))
time.sleep(2)
ts = timed(fwd, 20)
print("after 2 s idle: %.3f ms" % (sum(ts) / 20))
la2.la2_backward(q, k, v, do, dec); torch.cuda.synchronize()
ts = timed(fwd, 20)
print("right after one bwd: %.3f ms" % (sum(ts) / 20))
time.sleep(2)
ts = timed(fwd, 20)
print("after bwd + 2 s idle: %.3f ms" % (sum(ts) / 20))
step = lambda: (la2.la2_forward(q, k, v, dec), la2.la2_backward(q, k, v, do, dec))
ts = timed(step, 100)
print("step x100: first 5 %.3f, last 5 %.3f ms" % (sum(ts[:5]) / 5, sum(ts[-5:]) / 5))
