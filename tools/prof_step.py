"""Run a few fwd+bwd steps of the C2 shape for ncu captures (not a benchmark)."""
import argparse, sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
ap = argparse.ArgumentParser()
ap.add_argument('--seq-len', type=int, default=8192)
ap.add_argument('--batch', type=int, default=8)
ap.add_argument('--heads', type=int, default=16)
ap.add_argument('--dim', type=int, default=64)
ap.add_argument('--steps', type=int, default=3)
a = ap.parse_args()
dev = torch.device('cuda', 0)
B, H, N, D = a.batch, a.heads, a.seq_len, a.dim
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
from paper_2401_04658_b200 import ops
stored = ops.STORED_STATES and D == 64 and N >= ops.STORED_STATES_MIN_N  # as bench.py / autograd
for _ in range(a.steps):
    if stored:
        _, _, blocks = ops.la2_forward_states(q, k, v, dec)
        ops.la2_backward_states(q, k, v, do, dec, blocks)
    else:
        la2.la2_forward(q, k, v, dec)
        la2.la2_backward(q, k, v, do, dec)
torch.cuda.synchronize()
print('done')
