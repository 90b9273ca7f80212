"""Host link bandwidth: H2D, D2H, both at once, with 1 or 2 streams per direction (pinned)."""
import time
import torch

dev = torch.device("cuda", 0)
n = 1 << 30  # bytes per buffer
H = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(4)]
D = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(4)]
for t in H:
    t.fill_(1)


def run(up_streams, down_streams, reps=3):
    ss_up = [torch.cuda.Stream() for _ in range(up_streams)]
    ss_dn = [torch.cuda.Stream() for _ in range(down_streams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        for i, s in enumerate(ss_up):
            with torch.cuda.stream(s):
                for j in range(i, 2, up_streams):
                    D[j].copy_(H[j], non_blocking=True)
        for i, s in enumerate(ss_dn):
            with torch.cuda.stream(s):
                for j in range(i, 2, down_streams):
                    H[2 + j].copy_(D[2 + j], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    up = 2 * n if up_streams else 0
    dn = 2 * n if down_streams else 0
    return (up + dn) / dt / 1e9, up / dt / 1e9, dn / dt / 1e9


for cfg in [(1, 0), (2, 0), (0, 1), (0, 2), (1, 1), (2, 2)]:
    run(*cfg, reps=1)
    tot, up, dn = run(*cfg)
    print(f"up streams {cfg[0]} down streams {cfg[1]}: total {tot:.1f} GB/s (up {up:.1f}, down {dn:.1f})", flush=True)
