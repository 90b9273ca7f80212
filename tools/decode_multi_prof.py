"""One la2_decode_tokens launch (batch B, H=20, d=dv=128, T tokens) for ncu:
ncu --set full -k regex:decode_vec python tools/decode_multi_prof.py 256 8"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2401_04658_b200 as la2  # noqa: E402

B, T = int(sys.argv[1]), int(sys.argv[2])
H, D = 20, 128
dev = torch.device("cuda")
dec = la2.decay_tensor([0.9 + 0.005 * i for i in range(H)], H, dev)
st = torch.zeros(B, H, D, D, device=dev)
q, k, v = (torch.randn(B, H, T, D, device=dev).to(torch.bfloat16) for _ in range(3))
for _ in range(3):
    la2.decode_tokens(q, k, v, dec, st)
torch.cuda.synchronize()
