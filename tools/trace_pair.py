"""Phase trace of CTA (0,0,0) of the dK/dV cluster pair (the last tcgen05 launch of la2_backward)."""
import ctypes, os, sys
os.environ.setdefault('LA2_LIB', os.path.join(os.path.dirname(__file__), '..', 'paper_2401_04658_b200', 'libla2_trace.so'))
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200 import _lib
from bench import alibi_decay
lib = _lib.load()
la2.set_tuning(la2.ops.TUNE_CONCURRENT_BWD, 0)
la2.set_tuning(la2.ops.TUNE_PARTITION_BWD, 0)
lib.la2_set_trace.argtypes = [ctypes.c_void_p]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 8
H = int(sys.argv[4]) if len(sys.argv) > 4 else 16
N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
D = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device('cuda', 0)
q, k, v = ((torch.rand(B, H, N, D, device=dev) * 2 - 1).bfloat16() for _ in range(3))
dec = la2.decay_tensor(alibi_decay(H), H, dev)
buf = torch.zeros(4 * 64 * 8, dtype=torch.int64, device=dev)
TRIPLE = os.environ.get("TRACE_TRIPLE") == "1"  # the stored-state dQ/dK/dV triple instead
if TRIPLE:
    _, _, blocks = la2.ops.la2_forward_states(q, k, v, dec)
    bwd = lambda: la2.ops.la2_backward_states(q, k, v, q, dec, blocks)  # noqa: E731
else:
    bwd = lambda: la2.la2_backward(q, k, v, q, dec)  # noqa: E731
bwd()
lib.la2_set_trace(buf.data_ptr())
bwd()
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(4, 64, 8).astype(np.int64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1)
names = {0: "TMA  [pre-wait, loads]", 1: "MMA  [iter, S(i+1) issued, PREADY, OEMPTY, KVREADY, KT/DKVEMPTY, end]",
         2: "ROW  [A start, S ready, A end, B start, stbar, OFULL, B end]", 3: "STATE[K~ start, K ready, K~ end, U start, DKVFULL, U end, dkv loaded, OEFULL]"}
for role in range(4):
    print(names[role])
    for i in list(range(0, 4)) + list(range(40, 46)):
        print(f"  blk {i:3d}: " + " ".join(f"{x:8d}" for x in t[role, i] if x >= 0))
per = np.diff(t[2, 30:60, 0]).mean()
print("steady-state cycles per block (row A start):", per, "D =", D)
