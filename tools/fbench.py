"""Quick kernel timing for development: fwd / bwd ms and achieved GB/s per shape."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay

def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

if __name__ == "__main__":
    shapes = [(8, 16, 65536, 64), (8, 16, 8192, 64), (8, 16, 1024, 64), (2, 16, 16384, 128), (4, 20, 16384, 128)]
    if len(sys.argv) > 1:
        shapes = [tuple(map(int, s.split(','))) for s in sys.argv[1:]]
    dev = torch.device('cuda', 0)
    for B, H, N, D in shapes:
        q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
        dec = la2.decay_tensor(alibi_decay(H), H, dev)
        f = t(lambda: la2.la2_forward(q, k, v, dec))
        bw = t(lambda: la2.la2_backward(q, k, v, do, dec))
        fb = B * H * N * D * 2 * 4
        print(f"B={B} H={H} N={N} d={D}: fwd {f:.3f} ms ({fb / f / 1e6:.0f} GB/s)  bwd {bw:.3f} ms  "
              f"step {f + bw:.3f} ms  {B * N / (f + bw) / 1e3:.1f} Mtok/s", flush=True)
        del q, k, v, do
