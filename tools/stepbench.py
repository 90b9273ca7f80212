"""Development timing of one training step as the autograd entry point runs it
(ops.LightningAttn2Fn's policy: d = 64 with N >= STORED_STATES_MIN_N stores the forward's
per-block states and runs the dQ/dK/dV triple, otherwise forward + replaying backward).
Prints fwd / bwd / step ms per shape "B,H,N,d" (burst: rested GPU, 10 reps)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2401_04658_b200 as la2  # noqa: E402
from bench import alibi_decay  # noqa: E402
from paper_2401_04658_b200 import ops  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main(shapes, reps=10):
    dev = torch.device("cuda", 0)
    for B, H, N, D in shapes:
        q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
        dec = la2.decay_tensor(alibi_decay(H), H, dev)
        stored = ops.STORED_STATES and D == 64 and N >= ops.STORED_STATES_MIN_N
        if stored:
            _, _, blocks = ops.la2_forward_states(q, k, v, dec)
            f = timed(lambda: ops.la2_forward_states(q, k, v, dec), reps)
            bw = timed(lambda: ops.la2_backward_states(q, k, v, do, dec, blocks), reps)
        else:
            f = timed(lambda: la2.la2_forward(q, k, v, dec), reps)
            bw = timed(lambda: la2.la2_backward(q, k, v, do, dec), reps)
        print(f"B={B} H={H} N={N} d={D} {'stored' if stored else 'replay'}: fwd {f:.3f} ms  bwd {bw:.3f} ms  "
              f"step {f + bw:.3f} ms  {B * N / (f + bw) / 1e3:.1f} Mtok/s", flush=True)
        del q, k, v, do


if __name__ == "__main__":
    args = sys.argv[1:] or ["8,16,65536,64", "8,16,16384,64", "8,16,4096,64"]
    main([tuple(map(int, s.split(","))) for s in args])
