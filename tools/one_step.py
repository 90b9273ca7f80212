"""One forward + one backward at a given shape (for ncu captures)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
B, H, N, D = (tuple(map(int, sys.argv[1].split(','))) if len(sys.argv) > 1 else (8, 16, 16384, 64))
dev = torch.device('cuda', 0)
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
la2.la2_forward(q, k, v, dec)
la2.la2_backward(q, k, v, do, dec)
torch.cuda.synchronize()
