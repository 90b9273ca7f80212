"""Forward time vs the address placement of the output buffer (development)."""
import sys
sys.path.insert(0, '.')
import torch
import bench
import paper_2401_04658_b200 as la2
from tools.fbench import t
dev = torch.device('cuda', 0)
B, H, N, D = 8, 16, 65536, 64
dec = la2.decay_tensor(bench.alibi_decay(H), H, dev)
q, k, v, do = [(torch.rand(B, H, N, D, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(4)]
G = 1 << 30
base = q.data_ptr()
print("q k v do offsets (MiB):", [(x.data_ptr() - base) / 2**20 for x in (q, k, v, do)])
# place o at controlled offsets from a big arena
arena = torch.empty(12 * G + 64 * 2**20, dtype=torch.uint8, device=dev)
a0 = arena.data_ptr()
print("arena offset (MiB):", (a0 - base) / 2**20)
from paper_2401_04658_b200 import _lib, ops
def fwd_into(o):
    _lib.call("la2_forward", ops._ptr(q), ops._ptr(k), ops._ptr(v), ops._ptr(dec), o, None, None,
              B, H, N, D, D, 0, ops._stream(dev))
for shift_mb in [0, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 1536, 2048 + 2]:
    optr = a0 + shift_mb * 2**20
    optr = (optr + 2**21 - 1) // 2**21 * 2**21
    ms = t(lambda: fwd_into(optr), 20)
    print(f"o at arena+{shift_mb} MiB (o-q = {(optr - base) / 2**20:.0f} MiB, mod 1GiB {((optr - base) % G) / 2**20:.0f} MiB): fwd {ms:.3f} ms")
