"""One C5 fwd+bwd step (B=1 H=16 N=512K d=128, intra-GPU split) for ncu launch lists."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
dev = torch.device('cuda', 0)
H, D, N = 16, 128, 524288
q, k, v, do = ((torch.rand(1, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
for _ in range(2):
    qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
    o = la2.lightning_attn2(qg, kg, vg, dec)
    o.backward(do)
torch.cuda.synchronize()
