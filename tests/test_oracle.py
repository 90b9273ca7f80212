"""Pin the CPU oracle (oracle/tila_port.py) to the reference.

Two kinds of pins:
  * known-answer values copied from the reference's own test-suite
    (pkg/tests/test_reference.py, pkg/tests/test_kernel.py), and
  * golden vectors produced by running the reference itself
    (tests/golden/make_golden.py -> golden.npz).
CPU only.
"""

import numpy as np
import pytest


def proj(a, tag):
    a = np.asarray(a, np.float64)
    w = np.random.default_rng([7919, tag, a.shape[0], a.shape[1]]).standard_normal((16, a.size))
    return w @ a.ravel()


# ------------------------------------------------------------ known answers
def test_decay_mask_kat(port):
    # pkg/tests/test_reference.py:27-34
    assert port.decay_mask(3, 0.5).tolist() == [[1.0, 0.0, 0.0], [0.5, 1.0, 0.0], [0.25, 0.5, 1.0]]
    assert port.decay_mask(2, 1.0).tolist() == [[1.0, 0.0], [1.0, 1.0]]
    assert port.decay_mask(1, 0.9).tolist() == [[1.0]]


@pytest.mark.parametrize("lam", [0.3, 0.5, 0.9, 0.999, 1.0])
@pytest.mark.parametrize("n", [1, 2, 5, 17])
def test_decay_mask_structure(port, n, lam):
    # pkg/tests/test_reference.py:36-47
    m = port.decay_mask(n, lam)
    assert np.array_equal(np.diag(m), np.ones(n))
    assert np.array_equal(np.triu(m, 1), np.zeros((n, n)))
    for s in range(n - 1):
        for t in range(s + 1):
            assert m[s + 1, t] == m[s, t] * lam


def test_power_table_flush(port):
    # pkg/tests/test_reference.py:56-60
    pows = port.power_table(0.5, 1200, np.float32)
    assert pows[0] == 1.0 and pows[-1] == 0.0
    assert not np.any((pows > 0) & (pows < np.finfo(np.float32).tiny))


def test_domain_errors(port):
    for lam in (0.0, -0.5, 1.5):
        with pytest.raises(ValueError):
            port.decay_mask(3, lam)
    with pytest.raises(ValueError):
        port.decay_mask(0, 0.5)
    with pytest.raises(ValueError):
        port.block_decay(0, 0.5)
    with pytest.raises(ValueError):
        port.oracle_forward(np.ones((2, 3)), np.ones((2, 4)), np.ones((2, 3)), 0.5)
    with pytest.raises(ValueError):
        port.oracle_forward(np.ones((2, 3)), np.ones((2, 3)), np.ones((3, 3)), 0.5)
    with pytest.raises(ValueError):
        port.chunked_forward(np.ones((8, 4)), np.ones((8, 4)), np.ones((8, 4)), 0.9, 4,
                             port.KvState.fresh(3, 4))


def test_block_decay_kat(port):
    # pkg/tests/test_kernel.py:31-50
    bd = port.block_decay(3, 0.5)
    assert bd.lambda_powers.tolist() == [0.5, 0.25, 0.125]
    assert bd.complement_powers.tolist() == [0.25, 0.5, 1.0]
    assert port.block_decay(1, 0.7).lambda_powers.tolist() == [0.7]
    assert port.block_decay(1, 0.7).complement_powers.tolist() == [1.0]
    assert port.block_decay(4, 1.0).lambda_powers.tolist() == [1.0] * 4
    for lam in (0.25, 0.5, 1.0):  # :52-56 exact for dyadic rates
        bd = port.block_decay(12, lam)
        assert np.all(bd.lambda_powers * bd.complement_powers == lam ** 12)


def test_forward_kats(port):
    # pkg/tests/test_reference.py:64-71, :94-97; pkg/tests/test_kernel.py:80-83
    assert port.oracle_forward([[2.0]], [[3.0]], [[4.0]], 0.7).tolist() == [[24.0]]
    ones = [[1.0], [1.0]]
    assert port.oracle_forward(ones, ones, ones, 0.5).ravel().tolist() == [1.0, 1.5]
    assert port.tiled_forward(ones, ones, ones, 0.5, 1)[0].ravel().tolist() == [1.0, 1.5]
    o, _ = port.recurrent_forward(np.ones((4, 1)), np.ones((4, 1)), np.ones((4, 1)), 1.0)
    assert o.ravel().tolist() == [1.0, 2.0, 3.0, 4.0]


def test_backward_kats(port):
    # pkg/tests/test_reference.py:168-179; pkg/tests/test_kernel.py:149-154
    g = port.oracle_backward([[2.0]], [[3.0]], [[4.0]], [[1.0]], 0.7)
    assert (g.dq.tolist(), g.dk.tolist(), g.dv.tolist()) == ([[12.0]], [[8.0]], [[6.0]])
    ones = [[1.0], [1.0]]
    g = port.oracle_backward(ones, ones, ones, ones, 1.0)
    assert g.dq.ravel().tolist() == [1.0, 2.0]
    assert g.dk.ravel().tolist() == [2.0, 1.0]
    assert g.dv.ravel().tolist() == [2.0, 1.0]
    g = port.tiled_backward(ones, ones, ones, ones, 0.5, 1)
    assert g.dq.ravel().tolist() == [1.0, 1.5]
    assert g.dk.ravel().tolist() == [1.5, 1.0]
    assert g.dv.ravel().tolist() == [1.5, 1.0]


def test_inference_step_kats(port):
    # pkg/tests/test_reference.py:124-138
    st = port.KvState.fresh(1, 1)
    o, st = port.inference_step([1.0], [1.0], [1.0], st, 0.5)
    assert o.tolist() == [1.0] and st.kv.tolist() == [[1.0]] and st.tokens_absorbed == 1
    o, st = port.inference_step([1.0], [1.0], [1.0], st, 0.5)
    assert o.tolist() == [1.5] and st.kv.tolist() == [[1.5]] and st.tokens_absorbed == 2


def test_single_block_equals_oracle_exactly(port):
    # pkg/tests/test_kernel.py:73-78 and :140-147
    q, k, v, d_out = port.case_inputs(12, 4, 4, 1)
    expected = port.oracle_forward(q, k, v, 0.9)
    for block in (12, 13, 50):
        assert np.array_equal(port.tiled_forward(q, k, v, 0.9, block)[0], expected)
    q, k, v, d_out = port.case_inputs(9, 3, 3, 10)
    go = port.oracle_backward(q, k, v, d_out, 0.9)
    gt = port.tiled_backward(q, k, v, d_out, 0.9, 9)
    for a in ("dq", "dk", "dv"):
        assert np.array_equal(getattr(gt, a), getattr(go, a))


def test_compare_semantics(port):
    # pkg/src/tila/verify.py:50-75: denominator from the reference argument
    r = port.compare([[1.0, 2.0]], [[1.0, 4.0]], 0.6)
    assert r.max_abs_error == 2.0 and r.max_rel_error == 0.5 and r.passed
    r = port.compare([[1.0, 4.0]], [[1.0, 2.0]], 0.6)
    assert r.max_rel_error == 1.0 and not r.passed
    assert port.compare([[0.0]], [[0.0]], 0.0).passed


# ------------------------------------------------------------- golden vectors
def _grid_cases(golden):
    meta = golden["grid/meta"]
    return [(i, int(m[0]), int(m[1]), int(m[2]), int(m[3]), float(m[4]), int(m[5]))
            for i, m in enumerate(meta)]


def test_golden_grid_against_reference(golden, port):
    """Every output of the port matches the reference's own outputs on a
    stratified subset of the normative grid (pkg/src/tila/verify.py:127-138)."""
    worst = 0.0
    for ci, n, d, dv, block, lam, seed in _grid_cases(golden):
        q, k, v, d_out = port.case_inputs(n, d, dv, seed)
        res = {"oracle_o": port.oracle_forward(q, k, v, lam),
               "recurrent_o": port.recurrent_forward(q, k, v, lam)[0]}
        o, st = port.tiled_forward(q, k, v, lam, block)
        res["tiled_o"], res["tiled_kv"] = o, st.kv
        state = port.KvState.fresh(d, dv)
        outs, start = [], 0
        for length in port.ragged_partition(n, seed):
            oc, state = port.chunked_forward(q[start:start + length], k[start:start + length],
                                             v[start:start + length], lam, block, state)
            outs.append(oc)
            start += length
        res["chunked_o"], res["chunked_kv"] = np.concatenate(outs), state.kv
        go = port.oracle_backward(q, k, v, d_out, lam)
        gt = port.tiled_backward(q, k, v, d_out, lam, block)
        res.update(oracle_dq=go.dq, oracle_dk=go.dk, oracle_dv=go.dv,
                   tiled_dq=gt.dq, tiled_dk=gt.dk, tiled_dv=gt.dv)
        for name, arr in res.items():
            ref = golden[f"grid/{ci}/{name}/proj"]
            got = proj(arr, ci)
            scale = max(np.max(np.abs(ref)), 1e-12)
            err = np.max(np.abs(got - ref)) / scale
            worst = max(worst, err)
            assert err <= 1e-12, (ci, name, err)
            key = f"grid/{ci}/{name}/full"
            if key in golden:
                assert np.array_equal(arr, golden[key]), (ci, name)
    assert worst <= 1e-12


def test_golden_gpu_case_against_reference(golden, port):
    """The fixture that pins the CUDA path: the port reproduces the reference's
    stored outputs on the same bf16-representable inputs."""
    import torch

    arrs = [torch.from_numpy(golden[f"gpu/{n}_bf16bits"]).view(torch.bfloat16).double().numpy()
            for n in ("q", "k", "v", "do")]
    decay = golden["gpu/decay"].astype(np.float64)
    decay = np.asarray([0.9, 0.999])  # stored as fp32; the reference ran with these doubles
    o, kv = port.bhnd_forward(*arrs[:3], decay, block=64)
    dq, dk, dv = port.bhnd_backward(*arrs, decay, block=64)
    for name, got in (("o", o), ("kv", kv), ("dq", dq), ("dk", dk), ("dv", dv)):
        ref = golden[f"gpu/{name}"].astype(np.float64)
        assert port.rel_err(got, ref) <= 1e-6, name


def test_golden_decode(golden, port):
    st = port.KvState.fresh(4, 3)
    for t in range(8):
        o, st = port.inference_step(golden["decode/q"][t], golden["decode/k"][t],
                                    golden["decode/v"][t], st, 0.8)
        assert np.array_equal(o, golden["decode/o"][t])
        assert np.array_equal(st.kv, golden["decode/kv"][t])


def test_ragged_partition_sums(port):
    for n in (1, 7, 100, 1000):
        for seed in range(4):
            parts = port.ragged_partition(n, seed)
            assert sum(parts) == n and min(parts) >= 1
