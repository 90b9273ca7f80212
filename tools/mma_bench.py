import sys
sys.path.insert(0, '.')
import torch
from paper_2401_04658_b200 import _lib
# (M, N, a_mode, b_mn, chains)  chains in {1,2,4}; 4 needs N <= 64
cfgs = [(128, 256, 0, 0, 1), (128, 128, 0, 0, 1), (128, 128, 0, 0, 2), (128, 64, 0, 1, 1), (128, 64, 0, 1, 2),
        (128, 64, 0, 1, 4), (128, 64, 2, 1, 1), (128, 64, 2, 1, 4), (128, 128, 2, 1, 2), (64, 64, 1, 1, 1),
        (64, 64, 1, 1, 4), (128, 64, 1, 1, 4), (128, 32, 0, 0, 4), (128, 16, 0, 0, 4)]
iters = 4096
for ctas in (1, 148):
    for M, N, am, bm, ch in cfgs:
        out = torch.zeros(ctas, dtype=torch.int64, device='cuda')
        for _ in range(2):
            _lib.call_dev("la2_bench_umma", M, N, am, bm | (ch << 1), iters, ctas, out.data_ptr(), 0)
        torch.cuda.synchronize()
        cyc = out.float().mean().item() / iters
        print(f"ctas={ctas} M={M} N={N} a_mode={am} b_mn={bm} chains={ch}: {cyc:.1f} cyc/mma  "
              f"{2 * M * N * 16 / cyc:.0f} flop/cyc/SM", flush=True)
