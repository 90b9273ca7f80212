"""Multi-token decode (la2_decode_tokens) vs single steps at the C4 decode shape.

python tools/decode_multi.py [batch]   -- H=20, d=dv=128, bf16 inputs, fp32 state.
Prints us per launch, tokens/s and the state+io bandwidth per T."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2401_04658_b200 as la2  # noqa: E402


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    H, D = 20, 128
    dev = torch.device("cuda")
    dec = la2.decay_tensor([0.9 + 0.005 * i for i in range(H)], H, dev)
    st = torch.zeros(B, H, D, D, device=dev)
    qd, kd, vd = (torch.randn(64, B, H, D, device=dev).to(torch.bfloat16) for _ in range(3))
    g = torch.cuda.CUDAGraph()
    la2.decode_step(qd[0], kd[0], vd[0], dec, st)
    with torch.cuda.graph(g):
        for t in range(64):
            la2.decode_step(qd[t], kd[t], vd[t], dec, st)
    ms = timed(g.replay, 5) / 64
    sb = B * H * D * D * 4 * 2
    print(f"single step (graph of 64): {ms * 1e3:.1f} us/token-step, {B / ms * 1e3 / 1e6:.2f} M tok/s, "
          f"state {sb / ms / 1e6:.0f} GB/s")
    for T in (1, 2, 4, 8, 16, 32, 64):
        q, k, v = (torch.randn(B, H, T, D, device=dev).to(torch.bfloat16) for _ in range(3))
        ms = timed(lambda: la2.decode_tokens(q, k, v, dec, st))
        nb = sb + 4 * B * H * T * D * 2
        print(f"T={T:3d}: {ms * 1e3:8.1f} us/launch  {B * T / ms * 1e3 / 1e6:7.2f} M tok/s  "
              f"{nb / ms / 1e6:6.0f} GB/s")


if __name__ == "__main__":
    main()
