"""tila adapter (fp64, the reference's default dtype) speed per call vs size: one head
tiled_forward / tiled_backward through paper_2401_04658_b200.tila_api (host arrays in and
out, as the reference API), and a 64-head batched_forward."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2401_04658_b200 import tila_api  # noqa: E402


def t(fn, reps=5):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


for n, d in ((2048, 64), (8192, 64), (8192, 128), (65536, 64)):
    q, k, v, do = (tila_api.random_matrix(n, d, 10 + i) for i in range(4))
    f = t(lambda: tila_api.tiled_forward(q, k, v, 0.9, 64))
    b = t(lambda: tila_api.tiled_backward(q, k, v, do, 0.9, 64))
    print(f"n={n} d={d} fp64 one head: tiled_forward {f:.2f} ms, tiled_backward {b:.2f} ms", flush=True)
heads = [(tila_api.random_matrix(8192, 64, 100 + i), tila_api.random_matrix(8192, 64, 200 + i),
          tila_api.random_matrix(8192, 64, 300 + i), 0.9) for i in range(64)]
print(f"batched_forward 64 heads n=8192 d=64: {t(lambda: tila_api.batched_forward(heads, 64), 2):.2f} ms")
