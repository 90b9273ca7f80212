"""Time lightning_attn2 fwd+bwd with explicit seq_split values (development)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from bench import alibi_decay
dev = torch.device('cuda', 0)
for B, H, N, D in [(4, 20, 16384, 128), (1, 16, 131072, 128), (8, 16, 65536, 64)]:
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16().requires_grad_() for _ in range(4))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    for g in (1, 2, 4, 8):
        if N % (g * 128):
            continue
        def step():
            o = la2.lightning_attn2(q, k, v, dec, seq_split=g)
            o.backward(do)
        for _ in range(3): step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(5): step()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        print(f"B={B} H={H} N={N} d={D} split={g}: {ms:.3f} ms  {B * N / ms / 1e3:.1f} Mtok/s", flush=True)
    del q, k, v, do
