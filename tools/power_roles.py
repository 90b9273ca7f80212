"""Board power and SM clock while ONE kind of launch runs back to back for ~2.5 s:
the C2 forward (storing states), the C2 backward triple, and a device-to-device copy
of the same bytes (an HBM-bound reference). Which launch sets the sustained power cap?"""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402

import paper_2401_04658_b200 as la2  # noqa: E402
from bench import alibi_decay  # noqa: E402
from paper_2401_04658_b200 import ops  # noqa: E402

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)
B, H, N, D = 8, 16, 65536, 64
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
_, _, blocks = ops.la2_forward_states(q, k, v, dec)
src = torch.empty(2 << 30, dtype=torch.uint8, device=dev)
dst = torch.empty_like(src)
roles = {
    "forward (states)": lambda: ops.la2_forward_states(q, k, v, dec),
    "backward triple": lambda: ops.la2_backward_states(q, k, v, do, dec, blocks),
    "d2d copy 2 GiB": lambda: dst.copy_(src),
}
for name, fn in roles.items():
    time.sleep(3)
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((nv.nvmlDeviceGetPowerUsage(h) / 1000, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            time.sleep(0.01)

    th = threading.Thread(target=sampler)
    th.start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.time()
    n = 0
    e0.record()
    while time.time() - t0 < 2.5:
        fn()
        n += 1
        if n % 20 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    tail = samples[len(samples) // 3:]
    p = sorted(s[0] for s in tail)
    c = sorted(s[1] for s in tail)
    print(f"{name:18s}: {e0.elapsed_time(e1) / n:.3f} ms/launch over {n}; power median {p[len(p) // 2]:.0f} W "
          f"max {p[-1]:.0f} W; SM clock median {c[len(c) // 2]} MHz", flush=True)
