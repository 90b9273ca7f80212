"""Where does the ~22 us host cost of one la2_forward call go? (development)"""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200 import _lib, ops
dev = torch.device('cuda', 0)
B, H, N, D = 8, 16, 1024, 64
q, k, v = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(3))
dec = la2.decay_tensor([0.9] * H, H, dev)
o = torch.empty_like(v)
lib = _lib.load()
def bench(name, fn, n=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:40s} {(t1 - t0) / n * 1e6:7.2f} us/call", flush=True)
bench("ctypes no-op (la2_version)", lambda: lib.la2_version())
args = (ops._ptr(q), ops._ptr(k), ops._ptr(v), ops._ptr(dec), ops._ptr(o), None, None, B, H, N, D, D, 0, ops._stream(dev))
bench("raw la2_forward (C side + launch)", lambda: lib.la2_forward(*args), 500)
bench("ops.la2_forward (python + C)", lambda: ops.la2_forward(q, k, v, dec), 500)
bench("torch.empty_like", lambda: torch.empty_like(v))
bench("ops._stream", lambda: ops._stream(dev))
bench("ops.decay_tensor (cuda)", lambda: ops.decay_tensor(dec, H, dev))
bench("_check_qkv", lambda: ops._check_qkv(q, k, v))
