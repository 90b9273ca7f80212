"""One forward + one backward at a given shape "B,H,N,d[,s]" (for ncu / compute-sanitizer);
",s" runs the stored-state pair la2_forward_states + la2_backward_states (the d = 64 dQ/dK/dV
triple) instead of la2_forward + la2_backward; ",t" runs the multi-token decode instead:
N tokens through la2_decode_tokens (bf16 and fp32, plus a single step) from a random state;
",f" fp32 inputs: the SIMT kernels, through the autograd entry point (sequence split) and raw."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
from paper_2401_04658_b200 import ops
spec = sys.argv[1].split(',') if len(sys.argv) > 1 else ['8', '16', '16384', '64']
B, H, N, D = map(int, spec[:4])
stored = len(spec) > 4 and spec[4] == 's'
normed = len(spec) > 4 and spec[4] == 'n'  # Norm(.) fused into the forward epilogue
tokens = len(spec) > 4 and spec[4] == 't'  # multi-token decode
fp32 = len(spec) > 4 and spec[4] == 'f'    # fp32 inputs: the SIMT kernels (+ the split path)
dev = torch.device('cuda', 0)
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).to(torch.float32 if fp32 else torch.bfloat16)
               for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
if tokens:
    for dt in (torch.bfloat16, torch.float32):
        st = torch.rand(B, H, D, D, device=dev)
        la2.decode_tokens(q.to(dt), k.to(dt), v.to(dt), dec, st)
        la2.decode_step(q[:, :, 0].to(dt), k[:, :, 0].to(dt), v[:, :, 0].to(dt), dec, st)
elif fp32:
    qg, kg, vg = (t.clone().requires_grad_() for t in (q, k, v))
    la2.lightning_attn2(qg, kg, vg, dec).backward(do)   # split (chunk states, scans, carried passes)
    la2.la2_forward(q, k, v, dec)
    la2.la2_backward(q, k, v, do, dec)
elif normed:
    y, rstd, _, _ = ops.la2_forward_norm(q, k, v, dec, 1e-6, "head")
    dx = ops.rmsnorm_backward(do, y, rstd, "head")
    la2.la2_backward(q, k, v, dx, dec)
elif stored:
    _, _, blocks = ops.la2_forward_states(q, k, v, dec)
    ops.la2_backward_states(q, k, v, do, dec, blocks)
else:
    la2.la2_forward(q, k, v, dec)
    la2.la2_backward(q, k, v, do, dec)
torch.cuda.synchronize()
