import sys; sys.path.insert(0,'.')
import torch, paper_2401_04658_b200 as la2
from paper_2401_04658_b200 import ops
from bench import alibi_decay
dev=torch.device('cuda',0); B,H,N,D=8,16,65536,64
q,k,v,do=((torch.rand(B,H,N,D,device=dev)*2-1).bfloat16() for _ in range(4))
dec=la2.decay_tensor(alibi_decay(H),H,dev)
def t(fn,reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a,b=torch.cuda.Event(True),torch.cuda.Event(True); a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/reps
for i in range(2):
    print('plain fwd', round(t(lambda: la2.la2_forward(q,k,v,dec)),3), 'fused norm fwd', round(t(lambda: ops.la2_forward_norm(q,k,v,dec,1e-6,'head')),3),
      'unfused (fwd + rmsnorm)', round(t(lambda: ops.rmsnorm_forward(la2.la2_forward(q,k,v,dec)[0],1e-6,'head')),3), 'heads', round(t(lambda: ops.la2_forward_norm(q,k,v,dec,1e-6,'heads')),3), flush=True)
