"""Sustained fwd+bwd step time (mean of the last 50 of 150 steps) -- power-capped regime."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
dev = torch.device('cuda', 0)
shapes = [tuple(map(int, s.split(','))) for s in sys.argv[1:]] or [(8, 16, 65536, 64), (32, 16, 16384, 128)]
for B, H, N, D in shapes:
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    step = lambda: (la2.la2_forward(q, k, v, dec), la2.la2_backward(q, k, v, do, dec))
    n = 150
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    ev[0].record()
    for i in range(n):
        step(); ev[i + 1].record()
    torch.cuda.synchronize()
    ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(n)]
    print(f"B={B} H={H} N={N} d={D}: steps 5-15 {sum(ts[5:15]) / 10:.3f} ms, last 50 {sum(ts[-50:]) / 50:.3f} ms", flush=True)
    del q, k, v, do
    torch.cuda.synchronize()
    import time; time.sleep(3)
