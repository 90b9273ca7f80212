"""Small-N step rate: raw stream-ordered calls vs one CUDA graph of the same step
(B=8, H=16, d=64 bf16), plus host enqueue time per step. Prints one line per N."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2401_04658_b200 as la2  # noqa: E402
from paper_2401_04658_b200 import ops  # noqa: E402

B, H, D = 8, 16, int(sys.argv[1]) if len(sys.argv) > 1 else 64
SOAK = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0  # seconds of back-to-back steps first
dev = torch.device("cuda", 0)
decay = la2.decay_tensor([float(torch.exp(torch.tensor(-2.0 ** (-8 * (h + 1) / H)))) for h in range(H)], H, dev)


def step(q, k, v, do):
    if ops.STORED_STATES and D == 64 and q.shape[2] >= ops.STORED_STATES_MIN_N:
        _, _, blocks = ops.la2_forward_states(q, k, v, decay)
        ops.la2_backward_states(q, k, v, do, decay, blocks)
    else:
        la2.la2_forward(q, k, v, decay)
        la2.la2_backward(q, k, v, do, decay)


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    host = (time.perf_counter() - t0) / reps * 1e6
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, host


n = 1024
while n <= 65536:
    g = torch.Generator(device=dev).manual_seed(n)
    q, k, v, do = [(torch.rand(B, H, n, D, device=dev, generator=g) * 2 - 1).bfloat16() for _ in range(4)]
    reps = max(10, min(200, (1 << 23) // n))
    for _ in range(3):
        step(q, k, v, do)
    if SOAK:
        timed(lambda: step(q, k, v, do), max(4, int(SOAK * 1e3 / max(timed(lambda: step(q, k, v, do), 2)[0], 1e-3))))
    raw, host = timed(lambda: step(q, k, v, do), reps)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step(q, k, v, do)  # workspace for the capture stream
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        step(q, k, v, do)
    for _ in range(3):
        graph.replay()
    gr, ghost = timed(graph.replay, reps)
    print(f"N={n:6d} raw {raw*1e3:8.1f} us (host {host:6.1f} us) graph {gr*1e3:8.1f} us (host {ghost:5.1f})"
          f"  tok/s raw {B*n/raw/1e3:6.1f} M graph {B*n/gr/1e3:6.1f} M", flush=True)
    del q, k, v, do, graph
    torch.cuda.empty_cache()
    n *= 2
