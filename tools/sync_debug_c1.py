import sys, warnings
sys.path.insert(0, ".")
import torch
import paper_2401_04658_b200 as la2
dev = torch.device("cuda", 0)
B, H, N, D = 1, 8, 2048, 64
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1) for _ in range(4))
dec = la2.decay_tensor([0.5, 0.8, 0.9, 0.95, 0.99, 0.999, 0.9999, 1.0], H, dev)
def step():
    qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
    la2.lightning_attn2(qg, kg, vg, dec).backward(do)
for _ in range(3): step()
torch.cuda.synchronize()
torch.cuda.set_sync_debug_mode("warn")
warnings.simplefilter("always")
import traceback
def hook(message, category, filename, lineno, file=None, line=None):
    print("SYNC:", message)
    traceback.print_stack(limit=8)
warnings.showwarning = hook
step()
torch.cuda.synchronize()
print("done")
