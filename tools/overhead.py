"""Host-side launch overhead vs device time at small N (development)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
from tools.fbench import t
dev = torch.device('cuda', 0)
for N in (1024, 4096):
    B, H, D = 8, 16, 64
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    for name, fn in (("fwd", lambda: la2.la2_forward(q, k, v, dec)),
                     ("bwd", lambda: la2.la2_backward(q, k, v, do, dec))):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200): fn()
        cpu = (time.perf_counter() - t0) / 200 * 1e6
        torch.cuda.synchronize()
        gpu = t(fn, 50) * 1e3
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        gg = t(g.replay, 50) * 1e3
        print(f"N={N} {name}: host {cpu:.1f} us/call, stream-timed {gpu:.1f} us, graph-replayed {gg:.1f} us")
