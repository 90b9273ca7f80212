"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference ``tila`` package from /root/reference/pkg/src (read
only) and records its outputs into ``tests/golden/golden.npz``. The fixtures
travel with the repo; nothing at test time reads /root/reference.

Contents:
  grid/<i>/...   a stratified subset of the reference's normative equivalence
                 grid (pkg/src/tila/verify.py:127-138): 16 seeded random linear
                 functionals ("projections") of every output of oracle_forward,
                 recurrent_forward, tiled_forward (+ final state), chunked_forward
                 over ragged_partition (+ final state), oracle_backward and
                 tiled_backward; full arrays when n <= 16.
  gpu/...        one [B=1,H=2,N=160,d=64] case with bf16-representable inputs and
                 the reference's tiled fp64 outputs rounded to fp32, used to pin
                 the CUDA path directly to the reference.
  decode/...     eight inference_step outputs and states (pkg/src/tila/reference.py:162-181).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden.npz"
N_PROJ = 16


def projections(a: np.ndarray, tag: int) -> np.ndarray:
    """16 seeded random linear functionals of a matrix (float64)."""
    a = np.asarray(a, np.float64)
    w = np.random.default_rng([7919, tag, a.shape[0], a.shape[1]]).standard_normal((N_PROJ, a.size))
    return w @ a.ravel()


def grid_subset():
    import tila.verify as V

    cases = V.default_grid().cases
    # stratified: every 23rd case covers all n / d / dv / block / lam / seed values
    return cases[::23]


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    import tila
    from tila.verify import case_inputs, ragged_partition

    out: dict[str, np.ndarray] = {}
    cases = grid_subset()
    meta = []
    for ci, case in enumerate(cases):
        q, k, v, d_out = case_inputs(case, "double")
        res = {
            "oracle_o": tila.oracle_forward(q, k, v, case.lam),
            "recurrent_o": tila.recurrent_forward(q, k, v, case.lam)[0],
        }
        tf = tila.tiled_forward(q, k, v, case.lam, case.block)
        res["tiled_o"], res["tiled_kv"] = tf.o, tf.final_kv.kv
        state = tila.KvState.fresh(case.d, case.dv)
        outs, start = [], 0
        for length in ragged_partition(case.n, case.seed):
            o, state = tila.chunked_forward(q[start:start + length], k[start:start + length],
                                            v[start:start + length], case.lam, case.block, state)
            outs.append(o)
            start += length
        res["chunked_o"], res["chunked_kv"] = np.concatenate(outs), state.kv
        go = tila.oracle_backward(q, k, v, d_out, case.lam)
        gt = tila.tiled_backward(q, k, v, d_out, case.lam, case.block)
        res.update(oracle_dq=go.dq, oracle_dk=go.dk, oracle_dv=go.dv,
                   tiled_dq=gt.dq, tiled_dk=gt.dk, tiled_dv=gt.dv)
        for name, arr in res.items():
            out[f"grid/{ci}/{name}/proj"] = projections(arr, ci)
            if case.n <= 16:
                out[f"grid/{ci}/{name}/full"] = np.asarray(arr, np.float64)
        meta.append([case.n, case.d, case.dv, case.block, case.lam, case.seed])
    out["grid/meta"] = np.asarray(meta, np.float64)

    # direct GPU pin: bf16-representable inputs, reference tiled fp64 outputs
    import torch

    B, H, N, D = 1, 2, 160, 64
    decay = np.asarray([0.9, 0.999], np.float64)
    g = torch.Generator().manual_seed(2401)
    tens = [(torch.rand(B, H, N, D, generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(4)]
    arrs = [t.float().numpy().astype(np.float64) for t in tens]
    for name, t in zip(("q", "k", "v", "do"), tens):
        out[f"gpu/{name}_bf16bits"] = t.view(torch.int16).numpy()
    out["gpu/decay"] = decay.astype(np.float32)
    o = np.empty((B, H, N, D)); kv = np.empty((B, H, D, D))
    dq = np.empty_like(o); dk = np.empty_like(o); dv = np.empty_like(o)
    for h in range(H):
        q, k, v, do = (a[0, h] for a in arrs)
        tf = tila.tiled_forward(q, k, v, float(decay[h]), 64)
        o[0, h], kv[0, h] = tf.o, tf.final_kv.kv
        gb = tila.tiled_backward(q, k, v, do, float(decay[h]), 64)
        dq[0, h], dk[0, h], dv[0, h] = gb.dq, gb.dk, gb.dv
    for name, arr in (("o", o), ("kv", kv), ("dq", dq), ("dk", dk), ("dv", dv)):
        out[f"gpu/{name}"] = arr.astype(np.float32)

    # decode: eight inference steps at d=4, dv=3, lam=0.8
    rng = np.random.default_rng(99)
    st = tila.KvState.fresh(4, 3)
    qs, ks, vs = rng.uniform(-1, 1, (8, 4)), rng.uniform(-1, 1, (8, 4)), rng.uniform(-1, 1, (8, 3))
    os_, kvs = [], []
    for t in range(8):
        o_t, st = tila.inference_step(qs[t], ks[t], vs[t], st, 0.8)
        os_.append(o_t)
        kvs.append(st.kv.copy())
    out.update({"decode/q": qs, "decode/k": ks, "decode/v": vs, "decode/o": np.asarray(os_),
                "decode/kv": np.asarray(kvs)})

    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(cases)} grid cases)")


if __name__ == "__main__":
    main()
