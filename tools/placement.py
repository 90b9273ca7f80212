"""Forward time vs where the output buffer lives (development)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2401_04658_b200 as la2
from paper_2401_04658_b200 import _lib, ops
from tools.fbench import t
import bench
dev = torch.device('cuda', 0)
B, H, N, D = 8, 16, 65536, 64
dec = la2.decay_tensor(bench.alibi_decay(H), H, dev)
pre = torch.empty(B, H, N, D, dtype=torch.bfloat16, device=dev)          # allocated before q
q, k, v, do = [(torch.rand(B, H, N, D, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(4)]
post = torch.empty_like(q)                                                 # right after do
def fwd_into(o):
    _lib.call("la2_forward", ops._ptr(q), ops._ptr(k), ops._ptr(v), ops._ptr(dec), o.data_ptr(), None, None,
              B, H, N, D, D, 0, ops._stream(dev))
G = 1 << 30
def show(name, o):
    ms = t(lambda: fwd_into(o), 20)
    print(f"{name:28s} o-q = {(o.data_ptr() - q.data_ptr()) / 2**20:9.0f} MiB  fwd {ms:.3f} ms", flush=True)
show("pre (before q)", pre)
show("post (after do)", post)
show("do (alias, timing only)", do)
show("v (alias, timing only)", v)
dq, dk, dvv, _ = la2.la2_backward(q, k, v, do, dec)
torch.cuda.synchronize()
show("dq", dq); show("dk", dk); show("dv", dvv)
fresh = torch.empty_like(q)
show("fresh after bwd", fresh)
big = torch.empty(6 * G, dtype=torch.uint8, device=dev)
for off in (0, 2, 4, 6, 8, 64, 512, 1024, 3000):
    o = big[off * 2**20: off * 2**20 + G].view(torch.bfloat16).view(B, H, N, D)
    show(f"arena+{off}MiB", o)
