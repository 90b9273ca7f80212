"""Phase trace of CTA (0,0,0) of the fused backward kernel G (needs libla2_trace.so)."""
import ctypes, os, sys
os.environ['LA2_LIB'] = os.path.join(os.path.dirname(__file__), '..', 'paper_2401_04658_b200', 'libla2_trace.so')
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200 import _lib
from bench import alibi_decay
lib = _lib.load()
lib.la2_set_trace.argtypes = [ctypes.c_void_p]
B, H, N, D = 8, 16, int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 64
dev = torch.device('cuda', 0)
q, k, v, do = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
# run only G: trace buffer is shared by F (dQ pass) and G, so trace G alone via the ABI
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
buf = torch.zeros(5 * 64 * 8, dtype=torch.int64, device=dev)
la2.la2_backward(q, k, v, do, dec)
torch.cuda.synchronize()
lib.la2_set_trace(buf.data_ptr())
la2.la2_backward(q, k, v, do, dec)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(5, 64, 8).astype(np.int64)
names = {0: "TMA [pre, post EMPTY]", 1: "X [start, after FULL+SFREE]", 4: "Y [start, fold-ready, PREADY, KV+OEMPTY, end]",
         2: "ROW [A start, SFULL, A end, B start, OFULL, B end]", 3: "STATE [D start, D end, U start, DKVFULL, OFULL, U end]"}
# G trace stamps are later than F's: keep roles' values > F's max by using Y as reference
t0 = t[4][t[4] > 0].min()
for role in (0, 1, 4, 2, 3):
    print(names[role])
    for i in list(range(0, 3)) + list(range(40, 45)):
        print(f"  blk {i:3d}: " + " ".join(f"{x - t0:8d}" for x in t[role, i] if x > 0))
print("steady-state cycles per block (Y start):", np.diff(t[4, 30:60, 0]).mean())
