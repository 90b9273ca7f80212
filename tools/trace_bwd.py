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
buf = torch.zeros(5 * 64 * 8, dtype=torch.int64, device=dev)
la2.la2_backward(q, k, v, do, dec)
lib.la2_set_trace(buf.data_ptr())
la2.la2_backward(q, k, v, do, dec)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(5, 64, 8).astype(np.int64)
t0 = t[1:][t[1:] > 0].min()
t = np.where(t > 0, t - t0, -1)
names = {1: "X [start, FULL, SFREE, PREADY]", 4: "Y [start, dKV-ready, KVREADY, OEMPTY]",
         2: "ROW [A start, SFULL, A end, B pre, OFULLX, OEFULL, B end]", 3: "STATE [D start, D end, U start, DKVFULL, OEFULL, U end]"}
for role in (1, 4, 2, 3):
    print(names[role])
    for i in list(range(0, 3)) + list(range(40, 45)):
        print(f"  blk {i:3d}: " + " ".join(f"{x:8d}" for x in t[role, i] if x >= 0))
print("steady-state cycles per block (X start):", np.diff(t[1, 30:60, 0]).mean())
