"""Host overhead of the autograd entry point at small N: eager lightning_attn2 fwd+bwd vs
the same step through torch.cuda.make_graphed_callables (B=8 H=16 d=64 bf16)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2401_04658_b200 as la2  # noqa: E402
from bench import alibi_decay  # noqa: E402

B, H, D = 8, 16, 64
dev = torch.device("cuda", 0)
dec = la2.decay_tensor(alibi_decay(H), H, dev)
for N in (1024, 2048, 4096, 8192):
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    fn = lambda q_, k_, v_: la2.lightning_attn2(q_, k_, v_, dec)  # noqa: E731
    graphed = torch.cuda.make_graphed_callables(fn, tuple(t.clone().requires_grad_() for t in (q, k, v)))
    leaves = tuple(t.clone().requires_grad_() for t in (q, k, v))
    res = {}
    for name, f in (("eager", fn), ("graphed", graphed)):
        def step():
            o = f(*leaves)
            o.backward(do)
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        reps = 50
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        host = (time.perf_counter() - t0) / reps * 1e6
        torch.cuda.synchronize()
        res[name] = (e0.elapsed_time(e1) / reps * 1e3, host)
    print(f"N={N:5d}: eager {res['eager'][0]:7.1f} us/step (host {res['eager'][1]:6.1f} us)  graphed "
          f"{res['graphed'][0]:7.1f} us/step (host {res['graphed'][1]:6.1f} us)", flush=True)
