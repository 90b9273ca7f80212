"""One C5 step (single 512K sequence, H=16, d=128, intra-GPU split) for ncu launch lists."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
dev = torch.device('cuda', 0)
H, D, N = 16, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 524288
q, k, v, do = ((torch.rand(1, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
q.requires_grad_(); k.requires_grad_(); v.requires_grad_()
dec = la2.decay_tensor(alibi_decay(H), H, dev)
for _ in range(2):
    q.grad = k.grad = v.grad = None
    o = la2.lightning_attn2(q, k, v, dec)
    o.backward(do)
torch.cuda.synchronize()
print("split", la2.split_factor(1, H, N, D, D, torch.bfloat16))
