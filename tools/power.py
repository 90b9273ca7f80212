"""Power draw and clocks while fwd+bwd steps run back to back for ~3 s (development)."""
import sys, threading, time
sys.path.insert(0, '.')
import torch, pynvml as nv
import paper_2401_04658_b200 as la2
from bench import alibi_decay
nv.nvmlInit(); h = nv.nvmlDeviceGetHandleByIndex(0)
dev = torch.device('cuda', 0)
for (B, H, N, D) in [(8, 16, 65536, 64), (32, 16, 16384, 128)]:
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    samples, stop = [], threading.Event()
    def sampler():
        while not stop.is_set():
            samples.append((nv.nvmlDeviceGetPowerUsage(h) / 1000, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                            nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM), nv.nvmlDeviceGetTemperature(h, 0)))
            time.sleep(0.01)
    th = threading.Thread(target=sampler); th.start()
    t0 = time.time(); n = 0
    while time.time() - t0 < 3:
        la2.la2_forward(q, k, v, dec); la2.la2_backward(q, k, v, do, dec); n += 1
        if n % 20 == 0: torch.cuda.synchronize()
    torch.cuda.synchronize(); stop.set(); th.join()
    p = [s[0] for s in samples[len(samples)//3:]]
    print(f"d={D}: {n} steps in 3 s; power W median {sorted(p)[len(p)//2]:.0f} max {max(p):.0f}; "
          f"sm MHz {sorted(s[1] for s in samples)[len(samples)//2]}, mem MHz {samples[-1][2]}, temp {samples[-1][3]} C; "
          f"power limit {nv.nvmlDeviceGetEnforcedPowerLimit(h)/1000:.0f} W", flush=True)
    del q, k, v, do; torch.cuda.empty_cache(); time.sleep(3)
