"""CPU oracle: a NumPy restatement of the reference ``tila`` algorithms.

TEST INFRASTRUCTURE ONLY. This module is the checker for the CUDA path and the
CPU-baseline leg of ``bench.py``; nothing in the product package
(``paper_2401_04658_b200``) imports it. Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline / ``--impl reference``) may use it.

Parity pinning: every function here is checked against golden vectors produced
by the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/tila`` and records its outputs) and against the
known-answer values of the reference test-suite (``tests/test_oracle.py``).

Citations are to /root/reference/pkg/src/tila/<file>:<line>.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

REL_FLOOR = 1e-12  # verify.py:27


# --------------------------------------------------------------------------- types
@dataclass
class KvState:
    """Running d x dv state plus tokens absorbed (reference.py:21-30)."""

    kv: np.ndarray
    tokens_absorbed: int = 0

    @classmethod
    def fresh(cls, d: int, dv: int, dtype=np.float64) -> "KvState":
        return cls(np.zeros((d, dv), dtype), 0)


@dataclass
class GradBundle:
    """dq, dk, dv of <d_out, O> (reference.py:33-39)."""

    dq: np.ndarray
    dk: np.ndarray
    dv: np.ndarray


# ---------------------------------------------------------------- validation
def check_decay(lam: float) -> None:
    """reference.py:42-44: lam must lie in (0, 1]."""
    if not (0.0 < lam <= 1.0):
        raise ValueError(f"decay rate must be in (0, 1], got {lam}")


def _floatify(a) -> np.ndarray:
    """reference.py:47-51: non-float input is promoted to float64."""
    x = np.asarray(a)
    if x.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
        x = x.astype(np.float64)
    return x


def check_inputs(q, k, v, d_out=None):
    """reference.py:54-74: common dtype via result_type, 2-D, matching rows."""
    mats = [_floatify(q), _floatify(k), _floatify(v)]
    if d_out is not None:
        mats.append(_floatify(d_out))
    common = np.result_type(*mats)
    mats = [m.astype(common, copy=False) for m in mats]
    q, k, v = mats[0], mats[1], mats[2]
    if min(q.ndim, k.ndim, v.ndim) != 2 or max(q.ndim, k.ndim, v.ndim) != 2:
        raise ValueError("q, k, v must be 2-D matrices")
    if q.shape != k.shape:
        raise ValueError(f"q and k must have the same shape, got {q.shape} and {k.shape}")
    if v.shape[0] != q.shape[0]:
        raise ValueError(f"v must have {q.shape[0]} rows, got {v.shape[0]}")
    if d_out is None:
        return q, k, v
    if mats[3].shape != v.shape:
        raise ValueError(f"d_out must have shape {v.shape}, got {mats[3].shape}")
    return q, k, v, mats[3]


def check_block(block: int) -> None:
    """kernel.py:68-70."""
    if block < 1:
        raise ValueError(f"block must be >= 1, got {block}")


# ------------------------------------------------------------------ decay tables
def power_table(lam: float, count: int, dtype=np.float64) -> np.ndarray:
    """[lam^0 .. lam^(count-1)] by repeated multiplication in ``dtype``; entries
    after the first value below the dtype's smallest normal are exactly zero
    (reference.py:77-100)."""
    check_decay(lam)
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    dt = np.dtype(dtype)
    floor = np.finfo(dt).tiny
    step = dt.type(lam)
    table = np.zeros(count, dt)
    cur = dt.type(1.0)
    for idx in range(count):
        table[idx] = cur
        cur = cur * step
        if cur < floor:
            break
    return table


def decay_mask(n: int, lam: float, dtype=np.float64) -> np.ndarray:
    """Lower-triangular M[s,t] = lam^(s-t) (reference.py:103-115), built from
    the same power table so every consumer agrees bit for bit."""
    check_decay(lam)
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    pw = power_table(lam, n, dtype)
    s_idx, t_idx = np.indices((n, n))
    lag = s_idx - t_idx
    mask = np.where(lag >= 0, pw[np.clip(lag, 0, n - 1)], 0.0).astype(np.dtype(dtype))
    return mask


@dataclass
class BlockDecayDiag:
    """kernel.py:36-48: lambda_powers[j] = lam^(j+1), complement_powers[j] = lam^(B-1-j)."""

    lambda_powers: np.ndarray
    complement_powers: np.ndarray


def block_decay(block: int, lam: float, dtype=np.float64) -> BlockDecayDiag:
    """kernel.py:57-65."""
    check_block(block)
    pw = power_table(lam, block + 1, dtype)
    return BlockDecayDiag(pw[1:].copy(), pw[:block][::-1].copy())


# ----------------------------------------------------------------- quadratic oracle
def oracle_forward(q, k, v, lam: float) -> np.ndarray:
    """((q k^T) * M) v  (reference.py:118-132)."""
    q, k, v = check_inputs(q, k, v)
    check_decay(lam)
    weights = (q @ k.T) * decay_mask(q.shape[0], lam, q.dtype)
    return weights @ v


def oracle_backward(q, k, v, d_out, lam: float) -> GradBundle:
    """Full-mask analytic gradients (reference.py:184-204)."""
    q, k, v, d_out = check_inputs(q, k, v, d_out)
    check_decay(lam)
    m = decay_mask(q.shape[0], lam, q.dtype)
    a = (d_out @ v.T) * m
    p = (q @ k.T) * m
    return GradBundle(a @ k, a.T @ q, p.T @ d_out)


# -------------------------------------------------------------- per-token recurrence
def _token_step(state, lam_t, q_row, k_row, v_row):
    """reference.py:135-139: state' = lam*state + k v^T, read after the update."""
    nxt = lam_t * state
    nxt += np.outer(k_row, v_row)
    return q_row @ nxt, nxt


def recurrent_forward(q, k, v, lam: float):
    """reference.py:142-159."""
    q, k, v = check_inputs(q, k, v)
    check_decay(lam)
    dt = q.dtype
    lam_t = dt.type(lam)
    state = np.zeros((q.shape[1], v.shape[1]), dt)
    rows = np.empty((q.shape[0], v.shape[1]), dt)
    for t in range(q.shape[0]):
        rows[t], state = _token_step(state, lam_t, q[t], k[t], v[t])
    return rows, KvState(state, q.shape[0])


def inference_step(q_t, k_t, v_t, state: KvState, lam: float):
    """reference.py:162-181: one decode step, state not mutated."""
    check_decay(lam)
    qv = _floatify(q_t).ravel()
    kv_ = _floatify(k_t).ravel()
    vv = _floatify(v_t).ravel()
    cur = state.kv
    if cur.ndim != 2:
        raise ValueError("state.kv must be a 2-D matrix")
    d, dv = cur.shape
    if qv.shape[0] != d or kv_.shape[0] != d:
        raise ValueError(f"q_t and k_t must have length {d}, got {qv.shape[0]} and {kv_.shape[0]}")
    if vv.shape[0] != dv:
        raise ValueError(f"v_t must have length {dv}, got {vv.shape[0]}")
    dt = cur.dtype
    out, nxt = _token_step(cur, dt.type(lam), qv.astype(dt, copy=False), kv_.astype(dt, copy=False),
                           vv.astype(dt, copy=False))
    return out, KvState(nxt, state.tokens_absorbed + 1)


# ------------------------------------------------------------------- tiled passes
def _blocks(n: int, block: int):
    return [(a, min(a + block, n)) for a in range(0, n, block)]


class _Tables:
    """Per-pass decay tables sized by the block only (kernel.py:73-92)."""

    def __init__(self, n, lam, block, dt):
        diag = block_decay(block, lam, dt)
        self.row_read = diag.lambda_powers        # lam^(j+1)
        self.row_write = diag.complement_powers   # lam^(B-1-j)
        self.mask = decay_mask(min(block, n), lam, dt)
        self.block = block

    def write_weights(self, r):
        return self.row_write[self.block - r:]

    def fold(self, r):
        return self.row_read[r - 1]


def _scan_forward(q, k, v, tb: _Tables, state, out):
    """kernel.py:95-119: intra left product + inter read of the carried state."""
    for a, b in _blocks(q.shape[0], tb.block):
        r = b - a
        qb, kb, vb = q[a:b], k[a:b], v[a:b]
        local = (qb @ kb.T) * tb.mask[:r, :r]
        out[a:b] = local @ vb
        out[a:b] += (qb * tb.row_read[:r, None]) @ state
        scaled_k = kb * tb.write_weights(r)[:, None]
        state *= tb.fold(r)
        state += scaled_k.T @ vb
    return state


def tiled_forward(q, k, v, lam: float, block: int):
    """kernel.py:122-139; returns (o, KvState)."""
    q, k, v = check_inputs(q, k, v)
    check_decay(lam)
    check_block(block)
    dt = q.dtype
    tb = _Tables(q.shape[0], lam, block, dt)
    out = np.empty((q.shape[0], v.shape[1]), dt)
    state = _scan_forward(q, k, v, tb, np.zeros((q.shape[1], v.shape[1]), dt), out)
    return out, KvState(state, q.shape[0])


def chunked_forward(q, k, v, lam: float, block: int, state: KvState):
    """kernel.py:142-162: caller state copied, never mutated."""
    q, k, v = check_inputs(q, k, v)
    check_decay(lam)
    check_block(block)
    dt = q.dtype
    if state.kv.shape != (q.shape[1], v.shape[1]):
        raise ValueError(f"state.kv must have shape {(q.shape[1], v.shape[1])}, got {state.kv.shape}")
    tb = _Tables(q.shape[0], lam, block, dt)
    out = np.empty((q.shape[0], v.shape[1]), dt)
    carried = np.array(state.kv, dtype=dt, copy=True)
    carried = _scan_forward(q, k, v, tb, carried, out)
    return out, KvState(carried, state.tokens_absorbed + q.shape[0])


def tiled_backward(q, k, v, d_out, lam: float, block: int) -> GradBundle:
    """kernel.py:165-233: forward sweep for dq (state replayed), reverse sweep
    for dk/dv with the mirrored state folded after each block is emitted."""
    q, k, v, d_out = check_inputs(q, k, v, d_out)
    check_decay(lam)
    check_block(block)
    n, d = q.shape
    dvw = v.shape[1]
    dt = q.dtype
    tb = _Tables(n, lam, block, dt)
    dq = np.empty((n, d), dt)
    dk = np.empty((n, d), dt)
    dv = np.empty((n, dvw), dt)
    spans = _blocks(n, block)

    state = np.zeros((d, dvw), dt)
    for a, b in spans:
        r = b - a
        kb, vb, gb = k[a:b], v[a:b], d_out[a:b]
        local = (gb @ vb.T) * tb.mask[:r, :r]
        dq[a:b] = local @ kb
        dq[a:b] += (gb * tb.row_read[:r, None]) @ state.T
        scaled_k = kb * tb.write_weights(r)[:, None]
        state *= tb.fold(r)
        state += scaled_k.T @ vb

    mirror = np.zeros((d, dvw), dt)
    for a, b in reversed(spans):
        r = b - a
        qb, kb, vb, gb = q[a:b], k[a:b], v[a:b], d_out[a:b]
        w = tb.write_weights(r)[:, None]
        local = (gb @ vb.T) * tb.mask[:r, :r]
        dk[a:b] = local.T @ qb
        dk[a:b] += (vb * w) @ mirror.T
        local = (qb @ kb.T) * tb.mask[:r, :r]
        dv[a:b] = local.T @ gb
        dv[a:b] += (kb * w) @ mirror
        scaled_q = qb * tb.row_read[:r, None]
        mirror *= tb.fold(r)
        mirror += scaled_q.T @ gb
    return GradBundle(dq, dk, dv)


def batched_forward(inputs, block: int):
    """kernel.py:252-260 (sequential; per-head errors tagged as kernel.py:236-240)."""
    out = []
    for i, (q, k, v, lam) in enumerate(inputs):
        try:
            out.append(tiled_forward(q, k, v, lam, block))
        except Exception as exc:  # noqa: BLE001 - mirror the reference's re-raise
            raise type(exc)(f"head {i}: {exc}") from exc
    return out


def batched_backward(inputs, block: int):
    """kernel.py:263-266."""
    out = []
    for i, (q, k, v, d_out, lam) in enumerate(inputs):
        try:
            out.append(tiled_backward(q, k, v, d_out, lam, block))
        except Exception as exc:  # noqa: BLE001
            raise type(exc)(f"head {i}: {exc}") from exc
    return out


# --------------------------------------------------------------------- verify
@dataclass
class ErrorReport:
    max_abs_error: float
    max_rel_error: float
    location: tuple
    passed: bool
    label: str = ""


def compare(candidate, reference, tolerance: float, label: str = "") -> ErrorReport:
    """verify.py:50-75: worst |cand-ref| over max(max|ref|, 1e-12); the reference
    argument sets the denominator."""
    c = np.asarray(candidate, dtype=np.float64)
    r = np.asarray(reference, dtype=np.float64)
    if c.shape != r.shape:
        raise ValueError(f"shape mismatch: candidate {c.shape} vs reference {r.shape}")
    if c.size == 0:
        return ErrorReport(0.0, 0.0, (0, 0), True, label)
    gap = np.abs(c - r)
    flat = int(np.argmax(gap))
    where = np.unravel_index(flat, gap.shape)
    worst = float(gap.flat[flat])
    scale = max(float(np.max(np.abs(r))), REL_FLOOR)
    loc = (int(where[0]), int(where[1])) if len(where) == 2 else (int(where[0]), 0)
    return ErrorReport(worst, worst / scale, loc, worst / scale <= tolerance, label)


def rel_err(candidate, reference) -> float:
    return compare(candidate, reference, np.inf).max_rel_error


def random_matrix(rows: int, cols: int, seed: int, precision: str = "double") -> np.ndarray:
    """matrix.py:70-82: U[-1, 1] from default_rng(seed), cast to the precision."""
    if rows < 1 or cols < 1:
        raise ValueError(f"rows and cols must be >= 1, got {rows}x{cols}")
    if seed < 0:
        raise ValueError(f"seed must be a non-negative integer, got {seed}")
    dt = {"single": np.float32, "double": np.float64}[precision]
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(rows, cols)).astype(dt, copy=False)


def case_inputs(n, d, dv, seed, precision="double"):
    """verify.py:169-176: seeds 10*seed + {0: q, 1: k, 2: v, 3: d_out}."""
    base = 10 * int(seed)
    return (random_matrix(n, d, base, precision), random_matrix(n, d, base + 1, precision),
            random_matrix(n, dv, base + 2, precision), random_matrix(n, dv, base + 3, precision))


def ragged_partition(n: int, seed: int) -> list[int]:
    """verify.py:179-189."""
    gen = np.random.default_rng([seed, n])
    parts, left = [], n
    while left > 0:
        take = int(gen.integers(1, max(1, min(left, n // 3 + 1)) + 1))
        parts.append(take)
        left -= take
    return parts


def default_grid():
    """verify.py:127-138: (n, d, dv, block, lam, seed) cases of the normative grid."""
    return [(n, d, dv, blk, lam, seed)
            for n in (1, 2, 7, 16, 33, 64, 100, 256)
            for d in (1, 4, 32)
            for dv in (d, d + 3)
            for blk in (1, 4, 16, 64)
            for lam in (0.5, 0.9, 0.999, 1.0)
            for seed in (0, 1)]


# ------------------------------------------------------- batched [B,H,N,d] helpers
def bhnd_forward(q, k, v, decay, block=64, kv_in=None):
    """Apply tiled_forward per (b, h) of [B,H,N,d] arrays with per-head decay."""
    B, H, N, _ = q.shape
    out = np.empty(v.shape, np.result_type(q, v))
    states = np.empty((B, H, q.shape[3], v.shape[3]), out.dtype)
    for b in range(B):
        for h in range(H):
            st = KvState(np.zeros((q.shape[3], v.shape[3]), out.dtype) if kv_in is None
                         else np.asarray(kv_in[b, h], out.dtype))
            o, s = chunked_forward(q[b, h], k[b, h], v[b, h], float(decay[h]), block, st)
            out[b, h] = o
            states[b, h] = s.kv
    return out, states


def bhnd_backward(q, k, v, d_out, decay, block=64):
    """Apply tiled_backward per (b, h)."""
    B, H = q.shape[:2]
    dq = np.empty(q.shape, np.float64 if q.dtype == np.float64 else q.dtype)
    dk = np.empty_like(dq)
    dv = np.empty(v.shape, dq.dtype)
    for b in range(B):
        for h in range(H):
            g = tiled_backward(q[b, h], k[b, h], v[b, h], d_out[b, h], float(decay[h]), block)
            dq[b, h], dk[b, h], dv[b, h] = g.dq, g.dk, g.dv
    return dq, dk, dv


def bhnd_oracle_forward(q, k, v, decay):
    B, H = q.shape[:2]
    out = np.empty(v.shape, np.float64)
    for b in range(B):
        for h in range(H):
            out[b, h] = oracle_forward(q[b, h], k[b, h], v[b, h], float(decay[h]))
    return out


def bhnd_oracle_backward(q, k, v, d_out, decay):
    B, H = q.shape[:2]
    dq = np.empty(q.shape, np.float64)
    dk = np.empty(q.shape, np.float64)
    dv = np.empty(v.shape, np.float64)
    for b in range(B):
        for h in range(H):
            g = oracle_backward(q[b, h], k[b, h], v[b, h], d_out[b, h], float(decay[h]))
            dq[b, h], dk[b, h], dv[b, h] = g.dq, g.dk, g.dv
    return dq, dk, dv
