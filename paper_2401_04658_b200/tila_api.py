"""The reference's public operator API, re-targeted at the GPU kernels.

Same names, argument meaning and error behaviour as the reference ``tila``
package (pkg/src/tila/__init__.py:13-40), so the reference's own test suite runs
against this module (tests/test_gpu_reference_suites.py: 221 of its 222 tests pass; the
other asserts bitwise equality between inference_step and the reference's own
recurrent_forward, i.e. NumPy/OpenBLAS summation order -- it passes when
recurrent_forward is served from here too):

  tiled_forward(q, k, v, lam, block)            pkg/src/tila/kernel.py:122-139
  chunked_forward(q, k, v, lam, block, state)   pkg/src/tila/kernel.py:142-162
  tiled_backward(q, k, v, d_out, lam, block)    pkg/src/tila/kernel.py:165-233
  batched_forward(inputs, block, parallel)      pkg/src/tila/kernel.py:252-260
  batched_backward(inputs, block, parallel)     pkg/src/tila/kernel.py:263-266
  inference_step(q_t, k_t, v_t, state, lam)     pkg/src/tila/reference.py:162-181
  recurrent_forward(q, k, v, lam)               pkg/src/tila/reference.py:142-159
  random_matrix, save_fixture, load_fixture,    pkg/src/tila/matrix.py (re-exported from
  AttentionConfig, FixtureFormatError           ``matrix``: seeded inputs, text fixtures)

Inputs and outputs are 2-D NumPy arrays (one head), like the reference. The
arithmetic runs on the GPU in the reference's result dtype (np.result_type of the
inputs, reference.py:54-74): float64 inputs -- the reference's default -- on the
double-precision CUDA-core kernels (la2_*_f64), so the reference's own fp64 gates
(1e-10 .. 1e-12) hold through this adapter; float32 inputs on the fp32 kernels (the
north star's fp32 path, 1e-4 against the fp64 oracle). ``block`` is validated (>= 1,
kernel.py:68-70); the fp64 kernels tile by it (or its largest divisor <= 16), so, as in
the reference, chunks aligned to the block reproduce the one-call result bitwise; the
fp32 kernels choose their own tile (results are block-invariant up to rounding,
pkg/tests/test_kernel.py:97-102). ``parallel`` is accepted for signature
compatibility; all heads of a batched call run in one launch.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .matrix import (  # noqa: F401  (re-exported: the reference's top-level namespace)
    PRECISIONS,
    AttentionConfig,
    FixtureFormatError,
    dtype_for,
    load_fixture,
    precision_of,
    random_matrix,
    save_fixture,
)

_FLOATS = (np.dtype(np.float32), np.dtype(np.float64))


@dataclass
class KvState:
    """Running key-value summary plus tokens absorbed (reference.py:21-30)."""

    kv: np.ndarray
    tokens_absorbed: int = 0

    @classmethod
    def fresh(cls, d: int, dv: int, dtype=np.float64) -> "KvState":
        return cls(np.zeros((d, dv), dtype), 0)


@dataclass
class GradBundle:
    dq: np.ndarray
    dk: np.ndarray
    dv: np.ndarray


@dataclass
class TiledForwardResult:
    o: np.ndarray
    final_kv: KvState


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("tila_api runs on the GPU; no CUDA device is available (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _check_decay(lam: float) -> None:
    if not 0.0 < lam <= 1.0:
        raise ValueError(f"decay rate must be in (0, 1], got {lam}")


def _check_block(block: int) -> None:
    if block < 1:
        raise ValueError(f"block must be >= 1, got {block}")


def _as_float(a) -> np.ndarray:
    x = np.asarray(a)
    return x if x.dtype in _FLOATS else x.astype(np.float64)


def _check_inputs(q, k, v, d_out=None):
    """Validation and dtype promotion of pkg/src/tila/reference.py:54-74."""
    arrs = [_as_float(q), _as_float(k), _as_float(v)]
    if d_out is not None:
        arrs.append(_as_float(d_out))
    dt = np.result_type(*arrs)
    arrs = [a.astype(dt, copy=False) for a in arrs]
    q, k, v = arrs[:3]
    if q.ndim != 2 or k.ndim != 2 or v.ndim != 2:
        raise ValueError("q, k, v must be 2-D matrices")
    if q.shape != k.shape:
        raise ValueError(f"q and k must have the same shape, got {q.shape} and {k.shape}")
    if v.shape[0] != q.shape[0]:
        raise ValueError(f"v must have {q.shape[0]} rows, got {v.shape[0]}")
    if d_out is not None:
        if arrs[3].shape != v.shape:
            raise ValueError(f"d_out must have shape {v.shape}, got {arrs[3].shape}")
        return q, k, v, arrs[3]
    return q, k, v


def _tdt(dt) -> torch.dtype:
    """Device dtype for a reference result dtype: float64 stays float64."""
    return torch.float64 if np.dtype(dt) == np.float64 else torch.float32


def _dev(a: np.ndarray, dev, dt=np.float32) -> torch.Tensor:
    npdt = np.float64 if _tdt(dt) == torch.float64 else np.float32
    return torch.from_numpy(np.ascontiguousarray(a, dtype=npdt)).to(dev, non_blocking=False)


def _host(t: torch.Tensor, dt) -> np.ndarray:
    return t.detach().cpu().numpy().astype(dt, copy=False)


def _stack_heads(mats, dev, dt=np.float32):
    """list of H equal-shape 2-D arrays -> [1, H, n, c] on the device (fp64 for float64)."""
    return _dev(np.stack(mats)[None], dev, dt)


def tiled_forward(q, k, v, lam: float, block: int) -> TiledForwardResult:
    q, k, v = _check_inputs(q, k, v)
    _check_decay(lam)
    _check_block(block)
    [res] = _forward_group([(q, k, v, lam)], None, block)
    return res


def chunked_forward(q, k, v, lam: float, block: int, state: KvState):
    q, k, v = _check_inputs(q, k, v)
    _check_decay(lam)
    _check_block(block)
    d, dv = q.shape[1], v.shape[1]
    if state.kv.shape != (d, dv):
        raise ValueError(f"state.kv must have shape {(d, dv)}, got {state.kv.shape}")
    [res] = _forward_group([(q, k, v, lam)], [state.kv], block)
    return res.o, KvState(res.final_kv.kv, state.tokens_absorbed + q.shape[0])


def _forward_group(heads, states, block=0):
    """One launch for heads of identical shape; returns TiledForwardResult per head."""
    dev = _device()
    dt = np.result_type(*[h[0] for h in heads])
    qt = _stack_heads([h[0] for h in heads], dev, dt)
    kt = _stack_heads([h[1] for h in heads], dev, dt)
    vt = _stack_heads([h[2] for h in heads], dev, dt)
    kv_in = None if states is None else _stack_heads(list(states), dev, dt)
    o, kv = ops.la2_forward(qt, kt, vt, [float(h[3]) for h in heads], kv_in=kv_in,
                            output_final_state=True, block=block)
    o_h, kv_h = _host(o[0], dt), _host(kv[0], dt)
    n = heads[0][0].shape[0]
    return [TiledForwardResult(o_h[i], KvState(kv_h[i], n)) for i in range(len(heads))]


def tiled_backward(q, k, v, d_out, lam: float, block: int) -> GradBundle:
    q, k, v, d_out = _check_inputs(q, k, v, d_out)
    _check_decay(lam)
    _check_block(block)
    [g] = _backward_group([(q, k, v, d_out, lam)], block)
    return g


def _backward_group(heads, block=0):
    dev = _device()
    dt = np.result_type(*[h[0] for h in heads])
    q, k, v, do = (_stack_heads([h[j] for h in heads], dev, dt) for j in range(4))
    dq, dk, dv, _ = ops.la2_backward(q, k, v, do, [float(h[4]) for h in heads], block=block)
    dq, dk, dv = _host(dq[0], dt), _host(dk[0], dt), _host(dv[0], dt)
    return [GradBundle(dq[i], dk[i], dv[i]) for i in range(len(heads))]


def _batched(inputs, block, fn, ncheck):
    # per head, in the reference's order (inputs, decay, block: kernel.py:122-139), so an
    # error reads "head i: ..." and an empty input list returns [] whatever the block
    checked = []
    for i, item in enumerate(inputs):
        try:
            arrs = _check_inputs(*item[:ncheck])
            _check_decay(item[ncheck])
            _check_block(block)
        except Exception as exc:  # same re-raise as kernel.py:236-240
            raise type(exc)(f"head {i}: {exc}") from exc
        checked.append((*arrs, item[ncheck]))
    # group heads by shape and dtype so each group is one launch
    groups: dict = {}
    for i, h in enumerate(checked):
        groups.setdefault(tuple((a.shape, a.dtype) for a in h[:ncheck]), []).append(i)
    out = [None] * len(checked)
    for idxs in groups.values():
        for i, r in zip(idxs, fn([checked[i] for i in idxs])):
            out[i] = r
    return out


def batched_forward(inputs, block: int, parallel: bool = False) -> list[TiledForwardResult]:
    """Per-head forward with per-head decay; inputs is a list of (q, k, v, lam)."""
    return _batched(inputs, block, lambda hs: _forward_group(hs, None, block), 3)


def batched_backward(inputs, block: int, parallel: bool = False) -> list[GradBundle]:
    """Per-head backward; inputs is a list of (q, k, v, d_out, lam)."""
    return _batched(inputs, block, lambda hs: _backward_group(hs, block), 4)


def inference_step(q_t, k_t, v_t, state: KvState, lam: float):
    """One decode token; the input state is not modified (reference.py:162-181)."""
    _check_decay(lam)
    q_t, k_t, v_t = (_as_float(x).ravel() for x in (q_t, k_t, v_t))
    kv = state.kv
    if kv.ndim != 2:
        raise ValueError("state.kv must be a 2-D matrix")
    d, dv = kv.shape
    if q_t.shape[0] != d or k_t.shape[0] != d:
        raise ValueError(f"q_t and k_t must have length {d}, got {q_t.shape[0]} and {k_t.shape[0]}")
    if v_t.shape[0] != dv:
        raise ValueError(f"v_t must have length {dv}, got {v_t.shape[0]}")
    dev = _device()
    dt = kv.dtype  # the reference computes in the state's dtype (reference.py:178-180)
    st = _dev(kv, dev, dt).reshape(1, 1, d, dv).contiguous()
    o = ops.decode_step(_dev(q_t, dev, dt).reshape(1, 1, d), _dev(k_t, dev, dt).reshape(1, 1, d),
                        _dev(v_t, dev, dt).reshape(1, 1, dv), [float(lam)], st)
    return _host(o.reshape(dv), dt), KvState(_host(st.reshape(d, dv), dt), state.tokens_absorbed + 1)


def recurrent_forward(q, k, v, lam: float):
    """Per-token recurrent forward (reference.py:142-159) on the GPU decode kernels: one
    launch folds all n tokens through the recurrence (la2_decode_tokens[_f64]), each with
    inference_step's arithmetic, so folding :func:`inference_step` over the rows
    reproduces it bit for bit, as the reference's docstring promises."""
    q, k, v = _check_inputs(q, k, v)
    _check_decay(lam)
    n, d = q.shape
    dv = v.shape[1]
    dt = q.dtype
    if n == 0 or d == 0 or dv == 0:  # nothing to launch; the reference's values
        return np.zeros((n, dv), dt), KvState(np.zeros((d, dv), dt), n)
    dev = _device()
    o, st = ops.recurrent_forward(_dev(q, dev, dt)[None, None], _dev(k, dev, dt)[None, None],
                                  _dev(v, dev, dt)[None, None], [float(lam)])
    return _host(o[0, 0], dt), KvState(_host(st[0, 0], dt), n)
