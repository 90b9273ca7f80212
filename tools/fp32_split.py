"""fp32 C1 step time vs sequence split (development)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from tools.fbench import t
dev = torch.device('cuda', 0)
for (B, H, N, D) in [(1, 8, 2048, 64), (1, 8, 8192, 64), (1, 8, 1024, 64), (1, 1, 4096, 64), (1, 8, 2048, 128)]:
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1) for _ in range(4))
    dec = ([0.5, 0.8, 0.9, 0.95, 0.99, 0.999, 0.9999, 1.0] * 2)[:H]
    print(B, H, N, D, "auto split", la2.split_factor(B, H, N, D, D, torch.float32))
    for g in ["auto", 1, 4, 8, 16, 32, 64]:
        if g != "auto" and N % g:
            continue
        def step():
            qg, kg, vg = (x.detach().requires_grad_() for x in (q, k, v))
            o = la2.lightning_attn2(qg, kg, vg, dec, seq_split=g)
            o.backward(do)
        fw = t(lambda: la2.lightning_attn2(q, k, v, dec, seq_split=g))
        print(f"  split {g}: fwd {fw:.3f} ms  step {t(step):.3f} ms", flush=True)
