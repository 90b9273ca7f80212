"""Sustained (power-capped) step time of the C2 training step: 1 s soak, then 200 timed
steps; prints one line (for A/B of env knobs across processes)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2401_04658_b200 as la2  # noqa: E402
from bench import alibi_decay  # noqa: E402
from paper_2401_04658_b200 import ops  # noqa: E402

B, H, N, D = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,16,65536,64").split(","))
tag = sys.argv[2] if len(sys.argv) > 2 else ""
dev = torch.device("cuda", 0)
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
stored = ops.STORED_STATES and D == 64 and N >= ops.STORED_STATES_MIN_N


def step():
    if stored:
        _, _, blocks = ops.la2_forward_states(q, k, v, dec)
        ops.la2_backward_states(q, k, v, do, dec, blocks)
    else:
        la2.la2_forward(q, k, v, dec)
        la2.la2_backward(q, k, v, do, dec)


def timed(n):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


time.sleep(2)
burst = timed(10)
t0 = time.time()
while time.time() - t0 < 1.0:
    step()
torch.cuda.synchronize()
sus = timed(200)
print(f"{tag:12s} B={B} H={H} N={N} d={D}: burst {burst:.3f} ms  sustained {sus:.3f} ms "
      f"({B * N / sus / 1e3:.1f} M tok/s)", flush=True)
