"""Why is the forward slower after a backward? (development)"""
import sys
sys.path.insert(0, '.')
import torch
import bench
import paper_2401_04658_b200 as la2
from tools.fbench import t
dev = torch.device('cuda', 0)
B, H, N, D = 8, 16, 65536, 64
dec = la2.decay_tensor(bench.alibi_decay(H), H, dev)
q, k, v, do = [(torch.rand(B, H, N, D, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(4)]
f = lambda: la2.la2_forward(q, k, v, dec)
print("fwd fresh", t(f, 20))
x = torch.ones(3 * B * H * N * D, dtype=torch.bfloat16, device=dev)
print("fwd after 3GiB alloc", t(f, 20))
del x
torch.cuda.empty_cache()
print("fwd after free", t(f, 20))
la2.la2_backward(q, k, v, do, dec)
torch.cuda.synchronize()
print("fwd after 1 bwd", t(f, 20))
torch.cuda.empty_cache()
print("fwd after 1 bwd + empty_cache", t(f, 20))
print("bwd", t(lambda: la2.la2_backward(q, k, v, do, dec), 10))
print("fwd after bwds", t(f, 20))
la2.set_tuning(la2.ops.TUNE_PERSISTENT, 0)
print("bwd nonpersistent", t(lambda: la2.la2_backward(q, k, v, do, dec), 10))
print("fwd after nonpersistent bwds", t(f, 20))
torch.cuda.empty_cache()
print("fwd after empty_cache", t(f, 20))
o = torch.empty_like(v)
print("fwd with held o", t(f, 20))
