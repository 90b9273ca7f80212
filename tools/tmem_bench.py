import sys
sys.path.insert(0, '.')
import torch
from paper_2401_04658_b200 import _lib
iters = 4096
for warps in (4, 8, 16):
    for batch in (1, 4):
        ctas = 148
        out = torch.zeros(ctas, dtype=torch.int64, device='cuda')
        sink = torch.zeros(ctas * warps * 32, device='cuda')
        for _ in range(2):
            _lib.call_dev("la2_bench_tmem", warps, iters, batch, ctas, out.data_ptr(), sink.data_ptr(), 0)
        torch.cuda.synchronize()
        cyc = out.float().mean().item()
        total = warps * iters * 32 * 64  # bytes per SM
        print(f"warps={warps} batch={batch}: {total / cyc:.1f} B/cycle/SM  ({cyc / iters:.1f} cyc per ld16 per warp)", flush=True)
