"""State-only pass (chunk_state / chunk_dstate) timing at C5-like chunked shapes (development)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
from tools.fbench import t
dev = torch.device('cuda', 0)
for (B, H, N, D) in [(1, 128, 65536, 128), (1, 128, 65536, 64), (8, 16, 65536, 64)]:
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    dec = la2.decay_tensor(([0.999] * H), H, dev)
    ts = t(lambda: la2.chunk_state(k, v, dec))
    td = t(lambda: la2.chunk_dstate(q, do, dec))
    gb = 2 * B * H * N * D * 2 / 1e9
    print(f"B={B} H={H} N={N} d={D}: chunk_state {ts:.3f} ms ({gb / ts:.2f} TB/s)  chunk_dstate {td:.3f} ms ({gb / td:.2f} TB/s)", flush=True)
    del q, k, v, do
H, D, N = 16, 128, 524288
q, k, v, do = ((torch.rand(1, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
def step():
    qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
    o = la2.lightning_attn2(qg, kg, vg, dec)
    o.backward(do)
print(f"C5 step {t(step, 5):.3f} ms", flush=True)
