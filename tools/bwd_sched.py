"""Backward scheduling knobs vs N (development): default, no partition, no concurrency, no PDL."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200 import ops
from bench import alibi_decay
from tools.fbench import t
dev = torch.device('cuda', 0)
B, H, D = 8, 16, 64
base = {ops.TUNE_CONCURRENT_BWD: 16384, ops.TUNE_PARTITION_BWD: 8192, ops.TUNE_PDL: 4096}  # la2.h defaults
variants = {
    "default": {},
    "no-partition": {ops.TUNE_PARTITION_BWD: 0},
    "no-concurrency": {ops.TUNE_PARTITION_BWD: 0, ops.TUNE_CONCURRENT_BWD: 0},
    "no-pdl": {ops.TUNE_PDL: 0},
    "partition-32k": {ops.TUNE_PARTITION_BWD: 32768, ops.TUNE_CONCURRENT_BWD: 32768},
}
for N in (1024, 2048, 4096, 8192, 16384, 32768):
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    dec = la2.decay_tensor(alibi_decay(H), H, dev)
    row = []
    for name, kv in variants.items():
        for kk, vv in base.items():
            ops.set_tuning(kk, vv)
        for kk, vv in kv.items():
            ops.set_tuning(kk, vv)
        row.append(f"{name} {t(lambda: (la2.la2_forward(q, k, v, dec), la2.la2_backward(q, k, v, do, dec)), 20):.4f}")
    print(f"N={N}: " + " | ".join(row), flush=True)
    del q, k, v, do
