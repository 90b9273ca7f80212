import sys, threading, torch
sys.path.insert(0, '.')
import paper_2401_04658_b200 as la2
dev = torch.device('cuda', 0)
B, H, N, D = 1, 2, 300, 64
g = torch.Generator().manual_seed(0)
q, k, v, do = ((torch.rand(B, H, N, D, generator=g) * 2 - 1).bfloat16() for _ in range(4))
qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
for name, fn in [("fwd", lambda: la2.la2_forward(qd, kd, vd, [0.9, 1.0])),
                 ("bwd-main", lambda: la2.la2_backward(qd, kd, vd, dod, [0.9, 1.0]))]:
    try:
        fn(); torch.cuda.synchronize(); print(name, "ok")
    except Exception as e:
        print(name, "FAIL", e)
res = {}
def th():
    try:
        la2.la2_backward(qd, kd, vd, dod, [0.9, 1.0]); torch.cuda.synchronize(); res['t'] = 'ok'
    except Exception as e:
        res['t'] = f'FAIL {e}'
t = threading.Thread(target=th); t.start(); t.join(); print("bwd-thread", res)
