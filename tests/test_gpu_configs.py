"""GPU parity at the BASELINE configurations the bench runs:

  C3  B=32 H=16 N=16384 d=128   512 value-slice pair units over 74 clusters: the
                                 persistent stream-K schedule splits units across work
                                 ranges, so the fp32 state hand-off runs at long N
  C4  B=4  H=20 N=16384 d=128   80 pair units > 74 co-resident clusters
  C5  B=1  H=16 N=524288 d=128  one long sequence on one GPU: intra-GPU 8-way sequence
                                 split (chunk states, state scan, carried passes)
  C2 x4 B=8 H=16 N=262144 d=64  the headline shape at 4x the sequence: 2^31 elements per
                                 tensor (4 GiB bf16), so any 32-bit flat index overflows;
                                 the stored-state training path (forward states + triple)

Each runs the production entry point (``lightning_attn2`` forward + autograd backward)
on the full configuration and compares a subset of heads with the fp64 oracle port
(tiled, block 64; pinned to the reference by tests/test_oracle.py) on the same bf16
inputs, with the reference's metric (verify.py:50-75) and the north star's bf16
tolerance 1e-2. The head subset always includes lam = 1, 0.99999 and 0.9999 heads
(SURVEY.md:375): with those the carried state never decays away, so a broken carry
or hand-off cannot pass.
"""

import concurrent.futures as cf
import multiprocessing as mp

import pytest
import torch

import paper_2401_04658_b200 as la2

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2


def _oracle(args):
    q, k, v, do, lam = args
    from oracle import tila_port as port

    o, kv = port.tiled_forward(q, k, v, lam, 64)
    g = port.tiled_backward(q, k, v, do, lam, 64)
    return o, g.dq, g.dk, g.dv


def _rel(got, ref):
    from oracle import tila_port as port

    return port.rel_err(got, ref)


def run_config(B, H, N, D, decay, picks, seed=0):
    """fwd+bwd of the whole configuration on the GPU, then the picked (b, h) heads
    against the oracle. Returns {(b, h): {o, dq, dk, dv rel errors}}."""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    q, k, v, do = ((torch.rand(B, H, N, D, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
                   for _ in range(4))
    dec = torch.tensor(decay, dtype=torch.float32, device=dev)
    qg, kg, vg = (t.clone().requires_grad_() for t in (q, k, v))
    o = la2.lightning_attn2(qg, kg, vg, dec)
    o.backward(do)
    torch.cuda.synchronize()
    f64 = lambda t, b, h: t[b, h].detach().double().cpu().numpy()  # noqa: E731
    tasks, gots = [], []
    for b, h in picks:
        tasks.append((f64(q, b, h), f64(k, b, h), f64(v, b, h), f64(do, b, h), decay[h]))
        gots.append([f64(t, b, h) for t in (o, qg.grad, kg.grad, vg.grad)])
    del q, k, v, do, qg, kg, vg, o
    torch.cuda.empty_cache()
    with cf.ProcessPoolExecutor(max_workers=len(tasks), mp_context=mp.get_context("spawn")) as ex:
        refs = list(ex.map(_oracle, tasks))
    out = {}
    for (b, h), got, ref in zip(picks, gots, refs):
        out[(b, h, decay[h])] = {n: _rel(x, r) for n, x, r in zip(("o", "dq", "dk", "dv"), got, ref)}
    return out


def split_units(units, nblk, ranges):
    """Units whose blocks straddle a persistent work-range boundary (Sched in
    csrc/la2_tc_common.cuh: range c = [c*W/P, (c+1)*W/P) of the units x nblk space)."""
    W = units * nblk
    return sorted({(W * c // ranges) // nblk for c in range(1, ranges) if (W * c // ranges) % nblk})


# decay per head: near-1 heads where a broken carry would show, plus ordinary ones
C3_DECAY = [0.9999, 0.5, 0.9, 0.99, 0.999, 0.99999, 1.0, 0.95, 0.8, 0.999, 0.9999, 0.99999, 1.0,
            0.99, 0.9, 0.7]
C4_DECAY = [1.0, 0.99999, 0.9999, 0.999, 0.99, 0.9, 0.5, 0.8, 0.95, 0.999, 1.0, 0.99999, 0.9999,
            0.7, 0.9, 0.99, 0.3, 0.6, 0.999, 0.9999]
C5_DECAY = [1.0, 0.99999, 0.9999, 0.999, 0.99, 0.9, 0.5, 0.8, 0.95, 0.999, 1.0, 0.99999, 0.9999,
            0.7, 0.9, 0.99]


def test_split_units_helper():
    # C3: 512 pair units x 128 blocks over 74 clusters -> range 1 starts inside unit 6
    s = split_units(512, 128, 74)
    assert 6 in s and 262 in s and len(s) >= 60


def test_c3_parity():
    B, H, N, D = 32, 16, 16384, 128
    # pair units = (b, h) rows; 6 and 262 straddle a work-range boundary (stream-K hand-off)
    assert {6, 262} <= set(split_units(B * H, N // 128, 74))
    picks = [(0, 6), (16, 6), (0, 5), (0, 0), (31, 15), (20, 12)]
    errs = run_config(B, H, N, D, C3_DECAY, picks)
    print("C3 rel errors:", errs)
    assert {1.0, 0.99999, 0.9999} <= {lam for (_, _, lam) in errs}
    worst = max(max(e.values()) for e in errs.values())
    assert worst <= BF16_TOL, errs


def test_c4_parity():
    B, H, N, D = 4, 20, 16384, 128
    picks = [(0, 0), (0, 1), (0, 2), (1, 10), (3, 19), (2, 12)]
    errs = run_config(B, H, N, D, C4_DECAY, picks, seed=1)
    print("C4 rel errors:", errs)
    worst = max(max(e.values()) for e in errs.values())
    assert worst <= BF16_TOL, errs


def test_c5_one_gpu_parity():
    B, H, N, D = 1, 16, 524288, 128
    assert la2.split_factor(B, H, N, D, D, torch.bfloat16) == 8
    picks = [(0, 0), (0, 1), (0, 2)]  # lam = 1, 0.99999, 0.9999
    errs = run_config(B, H, N, D, C5_DECAY, picks, seed=2)
    print("C5 rel errors:", errs)
    worst = max(max(e.values()) for e in errs.values())
    assert worst <= BF16_TOL, errs


def test_c2_at_2g_elements_parity():
    B, H, N, D = 8, 16, 262144, 64
    assert B * H * N * D == 2 ** 31
    # the last head (highest addresses), the first, and the lam = 1 / 0.99999 heads
    picks = [(7, 15), (0, 0), (0, 6), (7, 5)]
    errs = run_config(B, H, N, D, C3_DECAY, picks, seed=3)
    print("C2 x4 rel errors:", errs)
    assert {1.0, 0.99999} <= {lam for (_, _, lam) in errs}
    worst = max(max(e.values()) for e in errs.values())
    assert worst <= BF16_TOL, errs
