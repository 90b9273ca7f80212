"""Does the d=128 backward time depend on where the tensors land? C3 shape, 8 placements
(each input carved at a random 4 KiB-multiple offset out of a larger buffer), 5 timed
backward calls each."""
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2401_04658_b200 as la2  # noqa: E402
from bench import alibi_decay  # noqa: E402

B, H, N, D = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,16,16384,128").split(","))
dev = torch.device("cuda", 0)
dec = la2.decay_tensor(alibi_decay(H), H, dev)
numel = B * H * N * D
rng = random.Random(0)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for trial in range(8):
    ts = []
    for _ in range(4):
        off = rng.randrange(0, 512) * 2048  # elements: 4 KiB multiples up to 2 MiB
        buf = torch.empty(numel + off, device=dev, dtype=torch.bfloat16)
        t = buf[off:off + numel].view(B, H, N, D)
        t.uniform_(-1, 1)
        ts.append(t)
    q, k, v, do = ts
    f = timed(lambda: la2.la2_forward(q, k, v, dec))
    bw = timed(lambda: la2.la2_backward(q, k, v, do, dec))
    print(f"trial {trial}: offsets(MiB) {[round((t.data_ptr() % (1 << 30)) / 2**20, 2) for t in ts]} "
          f"fwd {f:.3f} ms bwd {bw:.3f} ms", flush=True)
    del q, k, v, do, ts, buf
    torch.cuda.empty_cache()
