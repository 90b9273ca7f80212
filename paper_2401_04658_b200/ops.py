"""Torch-facing Lightning Attention-2 ops on the C ABI (``include/la2.h``).

``lightning_attn2(q, k, v, decay)`` is the drop-in entry point named by the
north star: q, k ``[B, H, N, d]``, v ``[B, H, N, dv]`` CUDA tensors (bf16 or
fp32), ``decay`` the per-head lambda in (0, 1]. Output
``o[b,h,t] = sum_{s<=t} lam_h^(t-s) (q_t . k_s) v_s`` -- exactly the
reference's ``oracle_forward`` / ``tiled_forward`` (pkg/src/tila/reference.py:118-132,
pkg/src/tila/kernel.py:122-139) applied per (b, h). No 1/sqrt(d) scale and no
Norm(.).

Every function here launches the CUDA kernels through ctypes on the current
torch stream; there is no CPU path.
"""

from __future__ import annotations

import ctypes
import weakref
from typing import Optional, Sequence, Union

import torch

from . import _lib

DecayLike = Union[float, Sequence[float], torch.Tensor]

# float64 runs the double-precision entry points (la2_*_f64, include/la2.h): the reference's
# default dtype, computed in fp64 as the reference does (no narrowing to fp32)
_DTYPE_CODE = {torch.bfloat16: _lib.LA2_BF16, torch.float32: _lib.LA2_FP32, torch.float64: -64}
_F64 = torch.float64


def _code(t: torch.Tensor) -> int:
    try:
        return _DTYPE_CODE[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}; expected torch.bfloat16, torch.float32 or "
                         "torch.float64") from None


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream(dev: torch.device) -> int:
    # raw handle of torch's current stream on dev (the C++ accessor; ~10x cheaper than
    # building a torch.cuda.Stream object per call)
    return torch._C._cuda_getCurrentRawStream(dev.index if dev.index is not None else
                                              torch.cuda.current_device())


def _on(device: torch.device, **tensors) -> None:
    """Every named tensor must be a CUDA tensor on ``device``: a host (or other-device)
    pointer reaching a kernel would fault and poison the CUDA context. There is no CPU path."""
    for name, t in tensors.items():
        if t is not None and (not t.is_cuda or t.device != device):
            raise ValueError(f"{name} must be a CUDA tensor on {device}, got one on {t.device}")


def decay_tensor(decay: DecayLike, H: int, device: torch.device, dtype=torch.float32) -> torch.Tensor:
    """Per-head decay as a contiguous float32 [H] tensor on ``device``.

    Values are validated with the reference's rule lam in (0, 1]
    (pkg/src/tila/reference.py:42-44) and raise ValueError otherwise: host values
    directly, a CUDA tensor through the C ABI's ``la2_check_decay`` once per
    (storage, version) -- the check synchronizes the stream, so repeated calls with
    the same unmodified tensor cost nothing after the first. Inside CUDA graph
    capture an unchecked tensor is not validated (the kernels turn an invalid lam
    into NaN outputs, never plausible numbers).
    """
    if isinstance(decay, torch.Tensor) and decay.is_cuda:
        if (decay.dtype == dtype and decay.dim() == 1 and decay.numel() == H
                and decay.device == device and decay.is_contiguous()):
            _check_cuda_decay(decay)
            return decay  # fast path: already a prepared per-head decay vector
        d = decay.to(device=device, dtype=dtype).reshape(-1)
        if d.numel() == 1:
            d = d.expand(H)
        if d.numel() != H:
            raise ValueError(f"decay must have {H} entries (one per head), got {d.numel()}")
        d = d.contiguous()
        _check_cuda_decay(d, decay)
        return d
    if isinstance(decay, torch.Tensor):
        vals = decay.detach().double().reshape(-1).tolist()
    elif isinstance(decay, (int, float)):
        vals = [float(decay)]
    else:
        vals = [float(x) for x in decay]
    if len(vals) == 1:
        vals = vals * H
    if len(vals) != H:
        raise ValueError(f"decay must have {H} entries (one per head), got {len(vals)}")
    for lam in vals:
        if not (0.0 < lam <= 1.0):
            raise ValueError(f"decay rate must be in (0, 1], got {lam}")
    return torch.tensor(vals, dtype=dtype, device=device)


_DECAY_CACHE: dict = {}
# tensor -> (data_ptr, version) last validated. Keyed by the tensor object (weakly): an
# address alone is not an identity -- the caching allocator hands a freed decay tensor's
# memory to the next one.
# (The map is by id() with a weak reference to confirm identity: tensors cannot be keys of
# a WeakKeyDictionary, whose lookups compare keys with the tensors' elementwise ==.)
_CHECKED: dict = {}


def _check_cuda_decay(d: torch.Tensor, src: Optional[torch.Tensor] = None) -> None:
    """la2_check_decay on a contiguous float32 CUDA decay vector ``d`` (derived from the
    caller's tensor ``src``, default ``d``), once per (tensor, version)."""
    owner = d if src is None else src
    stamp = (owner.data_ptr(), owner._version)
    hit = _CHECKED.get(id(owner))
    if hit is not None and hit[0]() is owner and hit[1] == stamp:
        return
    if torch.cuda.is_current_stream_capturing():
        return  # cannot synchronize inside capture; the kernels poison invalid lam with NaN
    _lib.call("la2_check_decay_f64" if d.dtype == _F64 else "la2_check_decay", d.data_ptr(), d.numel(),
              _stream(d.device))
    if len(_CHECKED) >= 4096:
        for key in [k for k, (r, _) in _CHECKED.items() if r() is None]:
            del _CHECKED[key]
    _CHECKED[id(owner)] = (weakref.ref(owner), stamp)


_REPEAT: dict = {}


def decay_repeat(dec: torch.Tensor, g: int) -> torch.Tensor:
    """``dec.repeat_interleave(g)`` for the g-way sequence split (head h's chunks are heads
    h*g .. h*g+g-1), cached per (validated decay tensor, version, g): the split path would
    otherwise build a fresh tensor per op, and a fresh CUDA decay tensor costs one
    validation -- a stream synchronization -- per call. The result inherits ``dec``'s
    validation."""
    key = (id(dec), g)
    stamp = (dec.data_ptr(), dec._version)
    hit = _REPEAT.get(key)
    if hit is not None and hit[0]() is dec and hit[1] == stamp:
        return hit[2]
    if dec.is_cuda:
        _check_cuda_decay(dec)
    r = dec.repeat_interleave(g)
    _CHECKED[id(r)] = (weakref.ref(r), (r.data_ptr(), r._version))
    if len(_REPEAT) >= 1024:
        for k_ in [k_ for k_, (w, _, _) in _REPEAT.items() if w() is None]:
            del _REPEAT[k_]
    _REPEAT[key] = (weakref.ref(dec), stamp, r)
    return r


def _decay(decay: DecayLike, H: int, device: torch.device, dtype=torch.float32) -> torch.Tensor:
    """decay_tensor for the ops' own use: host values (lists, floats, CPU tensors) are
    validated and uploaded once per distinct (values, device) and the device copy is
    reused -- a fresh upload costs ~16 us of host time per call. The cached tensor is
    never handed to the caller (only read by the kernels)."""
    if isinstance(decay, torch.Tensor) and decay.is_cuda:
        return decay_tensor(decay, H, device, dtype)
    if isinstance(decay, (int, float)):
        key = ((float(decay),), H, device, dtype)
    elif isinstance(decay, torch.Tensor):
        key = (tuple(decay.detach().double().reshape(-1).tolist()), H, device, dtype)
    else:
        key = (tuple(float(x) for x in decay), H, device, dtype)
    t = _DECAY_CACHE.get(key)
    if t is None:
        t = decay_tensor(list(key[0]), H, device, dtype)
        if len(_DECAY_CACHE) >= 256:
            _DECAY_CACHE.clear()
        _DECAY_CACHE[key] = t
    return t


def _check_qkv(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor):
    qs, vs = q.shape, v.shape
    if (len(qs) == 4 and k.shape == qs and len(vs) == 4 and vs[:3] == qs[:3] and q.is_cuda
            and q.dtype in _DTYPE_CODE and k.dtype == q.dtype and v.dtype == q.dtype
            and k.device == q.device and v.device == q.device):
        return qs[0], qs[1], qs[2], qs[3], vs[3]  # fast path (the common, valid call)
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise ValueError("q, k, v must be 4-D [B, H, N, d] tensors")
    if q.shape != k.shape:
        raise ValueError(f"q and k must have the same shape, got {tuple(q.shape)} and {tuple(k.shape)}")
    if v.shape[:3] != q.shape[:3]:
        raise ValueError(f"v must be [B, H, N, dv] matching q's {tuple(q.shape[:3])}, got {tuple(v.shape)}")
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise ValueError("q, k, v must be CUDA tensors (there is no CPU path)")
    if not (q.dtype == k.dtype == v.dtype):
        raise ValueError(f"q, k, v must share a dtype, got {q.dtype}, {k.dtype}, {v.dtype}")
    if not (q.device == k.device == v.device):
        raise ValueError("q, k, v must be on the same device")
    _code(q)
    B, H, N, d = q.shape
    return B, H, N, d, v.shape[3]


def _state(t: Optional[torch.Tensor], B, H, d, dv, device, name, dtype=torch.float32) -> Optional[torch.Tensor]:
    if t is None:
        return None
    if tuple(t.shape) != (B, H, d, dv):
        raise ValueError(f"{name} must have shape {(B, H, d, dv)}, got {tuple(t.shape)}")
    return t.to(device=device, dtype=dtype).contiguous()


# ------------------------------------------------------ intra-GPU sequence split
NUM_SMS = 148
def tc_shape(d: int, dv: int) -> bool:
    """bf16 widths on the tensor-core kernels (include/la2.h): d and dv multiples of 8 up to
    256 (d <= 128 padded to 64 / 128, d > 128 as split-d, dv in 64-wide slices)."""
    return 8 <= d <= 256 and d % 8 == 0 and 8 <= dv <= 256 and dv % 8 == 0
MAX_CHUNKS = 64  # la2_state_scan combines at most 64 chunk states per call


def split_factor(B: int, H: int, N: int, d: int, dv: int, dtype) -> int:
    """Chunks per sequence for the intra-GPU split (1 = no split).

    One CTA owns one (b, h, 64-wide value slice) for the whole sequence, so with
    fewer units than SMs the GPU idles. Viewing [B,H,N,d] as [B,H*G,N/G,d] (a free
    reshape) gives G x more units at the cost of one state-only pass over K,V (and
    Q,dO in the backward). Tensor-core path: used when units < ~100, chunks stay
    >= 8192 tokens and the split is at least 4-way (measured: at B=1, H=8, N=8192 the
    unsplit fwd+bwd takes 0.20 ms and every split 0.33-0.37 ms; at H=16, N=16384 splits
    are within noise of no split; at H=4, N=64K an 8-way split is 4.7x faster).
    SIMT path (fp32 / other shapes, several CTAs per SM): split until ~4 units per SM, down to 32-token chunks at d <= 64 (128 above), at most 64 chunks
    (the state scan's limit). Measured on B200 (tools/fp32_split.py): C1 fp32 fwd+bwd
    1.22 ms at 8 chunks -> 0.53 ms at 64.
    """
    if dtype == torch.float64:
        return 1  # the fp64 correctness path runs unsplit
    units = B * H * ((dv + 63) // 64)
    g = 1
    if dtype == torch.bfloat16 and tc_shape(d, dv):
        if units >= 100:
            return 1
        while (units * g < NUM_SMS and 2 * g <= MAX_CHUNKS and N % (2 * g * 128) == 0
               and N // (2 * g) >= 8192):
            g *= 2
        # each pass of a split runs over N/g tokens serially plus fixed launch/ramp costs,
        # so a 2-way split never pays (tools/bf16_split.py)
        return g if g >= 4 else 1
    if d > 256 or dv > 256:
        return 1
    min_chunk = 32 if max(d, dv) <= 64 else 128
    while units * g < 4 * NUM_SMS and 2 * g <= MAX_CHUNKS and N % (2 * g) == 0 and N // (2 * g) >= min_chunk:
        g *= 2
    return g


def _chunked(t: torch.Tensor, g: int) -> torch.Tensor:
    B, H, N, c = t.shape
    return t.view(B, H * g, N // g, c)


def _to_chunk_major(st: torch.Tensor, B: int, H: int, g: int) -> torch.Tensor:
    """[B, H*g, d, dv] -> [g, B, H, d, dv] (contiguous) for la2_state_scan."""
    d, dv = st.shape[-2:]
    return st.view(B, H, g, d, dv).permute(2, 0, 1, 3, 4).contiguous()


def _from_chunk_major(st: torch.Tensor, B: int, H: int, g: int) -> torch.Tensor:
    d, dv = st.shape[-2:]
    return st.permute(1, 2, 0, 3, 4).reshape(B, H * g, d, dv).contiguous()


def split_forward(q, k, v, decay, g: int, kv_in=None, output_final_state=False):
    """Forward with the sequence cut into g chunks per (b, h). Returns
    ``(o, kv_out, prefix)``; prefix (chunk-carried states) is reused by the backward."""
    B, H, N, d, dv = _check_qkv(q, k, v)
    dec = _decay(decay, H, q.device)
    dec_g = decay_repeat(dec, g)
    q4, k4, v4 = _chunked(q.contiguous(), g), _chunked(k.contiguous(), g), _chunked(v.contiguous(), g)
    s = chunk_state(k4, v4, dec_g)
    init = None if kv_in is None else _state(kv_in, B, H, d, dv, q.device, "kv_in")
    prefix = _from_chunk_major(state_scan(_to_chunk_major(s, B, H, g), dec, [N // g] * g, init=init), B, H, g)
    o4, kv4 = la2_forward(q4, k4, v4, dec_g, kv_in=prefix, output_final_state=output_final_state)
    kv_out = None if kv4 is None else kv4.view(B, H, g, d, dv)[:, :, -1].contiguous()
    return o4.view(B, H, N, dv), kv_out, prefix


def split_backward(q, k, v, d_out, decay, g: int, prefix, dkv_in=None, output_dkv=False):
    """Backward matching :func:`split_forward` (prefix = its chunk-carried states)."""
    B, H, N, d, dv = _check_qkv(q, k, v)
    _on(q.device, d_out=d_out)
    dec = _decay(decay, H, q.device)
    dec_g = decay_repeat(dec, g)
    q4, k4, v4, do4 = (_chunked(t.contiguous(), g) for t in (q, k, v, d_out))
    t = chunk_dstate(q4, do4, dec_g)
    init = None if dkv_in is None else _state(dkv_in, B, H, d, dv, q.device, "dkv_in")
    suffix = _from_chunk_major(state_scan(_to_chunk_major(t, B, H, g), dec, [N // g] * g, init=init,
                                          reverse=True), B, H, g)
    dq, dk, dvv, dkv4 = la2_backward(q4, k4, v4, do4, dec_g, kv_in=prefix, dkv_in=suffix,
                                     output_dkv=output_dkv)
    dkv_out = None if dkv4 is None else dkv4.view(B, H, g, d, dv)[:, :, 0].contiguous()
    return dq.view(B, H, N, d), dk.view(B, H, N, d), dvv.view(B, H, N, dv), dkv_out


# ------------------------------------------------------------------ raw passes
def la2_forward(q, k, v, decay: DecayLike, kv_in: Optional[torch.Tensor] = None,
                output_final_state: bool = False, block: int = 0):
    """One forward pass. Returns ``(o, kv_out)``; kv_out is None unless requested.

    kv_in (fp32 ``[B,H,d,dv]``, fp64 for fp64 inputs) is the carried state of
    tila.chunked_forward (pkg/src/tila/kernel.py:142-162); kv_out its returned KvState.kv.
    ``block`` (fp64 only) is the reference's block argument: the fp64 kernels tile by it
    (see include/la2.h la2_forward_f64); the bf16 / fp32 kernels choose their own tile.
    """
    B, H, N, d, dv = _check_qkv(q, k, v)
    if q.dtype == _F64:
        dec = _decay(decay, H, q.device, _F64)
        kv_in = _state(kv_in, B, H, d, dv, q.device, "kv_in", _F64)
        kv_out = torch.empty(B, H, d, dv, device=q.device, dtype=_F64) if output_final_state else None
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        o = torch.empty_like(v)
        _lib.call("la2_forward_f64", _ptr(q), _ptr(k), _ptr(v), _ptr(dec), _ptr(o), _ptr(kv_in), _ptr(kv_out),
                  B, H, N, d, dv, int(block), _stream(q.device))
        return o, kv_out
    dec = _decay(decay, H, q.device)
    kv_in = _state(kv_in, B, H, d, dv, q.device, "kv_in")
    kv_out = torch.empty(B, H, d, dv, device=q.device, dtype=torch.float32) if output_final_state else None
    lds = None
    if q.dtype == torch.bfloat16 and tc_shape(d, dv) and not (
            q.is_contiguous() and k.is_contiguous() and v.is_contiguous()):
        lds = [_head_stride(t) for t in (q, k, v)]
        if any(x is None for x in lds):
            lds = None
    if lds is not None:  # views (e.g. a chunk of a resident sequence): read in place
        o = torch.empty(B, H, N, dv, device=v.device, dtype=v.dtype)
        _lib.call("la2_forward_strided", _ptr(q), _ptr(k), _ptr(v), _ptr(dec), _ptr(o), _ptr(kv_in),
                  _ptr(kv_out), B, H, N, d, dv, _code(q), lds[0], lds[1], lds[2], _stream(q.device))
        return o, kv_out
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = torch.empty_like(v)
    _lib.call("la2_forward", _ptr(q), _ptr(k), _ptr(v), _ptr(dec), _ptr(o), _ptr(kv_in), _ptr(kv_out),
              B, H, N, d, dv, _code(q), _stream(q.device))
    return o, kv_out


def states_eligible(q: torch.Tensor, v: torch.Tensor) -> bool:
    """Shapes whose backward can use stored per-block states (la2_forward_states /
    la2_backward_states, include/la2.h): bf16, d = dv = 64."""
    return q.dtype == torch.bfloat16 and q.shape[3] == 64 and v.shape[3] == 64


def la2_forward_states(q, k, v, decay: DecayLike, kv_in: Optional[torch.Tensor] = None,
                       output_final_state: bool = False):
    """Forward that also returns the per-block bf16 states ``[B, H, ceil(N/128), d, dv]``
    (entry i = the state block i read: KV_{i-1}) for :func:`la2_backward_states`.
    Returns ``(o, kv_out, kv_blocks)``."""
    B, H, N, d, dv = _check_qkv(q, k, v)
    if not states_eligible(q, v):
        raise ValueError("stored per-block states need bf16 with d = dv = 64")
    dec = _decay(decay, H, q.device)
    kv_in = _state(kv_in, B, H, d, dv, q.device, "kv_in")
    kv_out = torch.empty(B, H, d, dv, device=q.device, dtype=torch.float32) if output_final_state else None
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = torch.empty_like(v)
    blocks = torch.empty(B, H, (N + 127) // 128, d, dv, device=q.device, dtype=torch.bfloat16)
    _lib.call("la2_forward_states", _ptr(q), _ptr(k), _ptr(v), _ptr(dec), _ptr(o), _ptr(kv_in),
              _ptr(kv_out), _ptr(blocks), B, H, N, d, dv, _code(q), _stream(q.device))
    return o, kv_out, blocks


def la2_backward_states(q, k, v, d_out, decay: DecayLike, kv_blocks: torch.Tensor, dkv_in=None,
                        output_dkv: bool = False):
    """Backward from the forward's stored per-block states (dQ without replaying the
    recurrence, in one 3-CTA cluster with the dK / dV reverse scans). Same results as
    :func:`la2_backward` up to rounding. Returns ``(dq, dk, dv, dkv_out)``."""
    B, H, N, d, dv = _check_qkv(q, k, v)
    if not states_eligible(q, v):
        raise ValueError("stored per-block states need bf16 with d = dv = 64")
    if d_out.shape != v.shape or d_out.dtype != v.dtype:
        raise ValueError(f"d_out must have shape {tuple(v.shape)} and dtype {v.dtype}")
    _on(q.device, d_out=d_out, kv_blocks=kv_blocks)
    nblk = (N + 127) // 128
    if (tuple(kv_blocks.shape) != (B, H, nblk, d, dv) or kv_blocks.dtype != torch.bfloat16
            or not kv_blocks.is_contiguous()):
        raise ValueError(f"kv_blocks must be a contiguous bf16 tensor of shape {(B, H, nblk, d, dv)}")
    dec = _decay(decay, H, q.device)
    dkv_in = _state(dkv_in, B, H, d, dv, q.device, "dkv_in")
    dkv_out = torch.empty(B, H, d, dv, device=q.device, dtype=torch.float32) if output_dkv else None
    q, k, v, d_out = q.contiguous(), k.contiguous(), v.contiguous(), d_out.contiguous()
    dq, dk, dvv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    _lib.call("la2_backward_states", _ptr(q), _ptr(k), _ptr(v), _ptr(d_out), _ptr(dec), _ptr(kv_blocks),
              _ptr(dq), _ptr(dk), _ptr(dvv), _ptr(dkv_in), _ptr(dkv_out), B, H, N, d, dv, _code(q),
              _stream(q.device))
    return dq, dk, dvv, dkv_out


# --------------------------------------------------------------------- Norm(.)
def _norm_group(norm: str, H: int) -> int:
    if norm == "head":
        return 1
    if norm == "heads":
        return H
    raise ValueError(f"norm must be None, 'head' (per head) or 'heads' (over all heads), got {norm!r}")


def rmsnorm_forward(x: torch.Tensor, eps: float = 1e-6, norm: str = "head", out: Optional[torch.Tensor] = None):
    """Norm(.) of NormAttention (an extension, SPEC.md:167 leaves it out):
    y = x / sqrt(mean(x^2) + eps) over each head's dv features ("head") or over all heads'
    features of a token ("heads"). Returns ``(y, rstd)``; ``out=x`` normalises in place."""
    B, H, N, dv = x.shape
    grp = _norm_group(norm, H)
    _on(x.device, x=x, out=out)
    x = x.contiguous()
    y = torch.empty_like(x) if out is None else out
    rstd = torch.empty(B, H // grp, N, device=x.device, dtype=torch.float32)
    _lib.call("la2_rmsnorm_forward", _ptr(x), _ptr(y), _ptr(rstd), B, H, N, dv, grp, float(eps), _code(x),
              _stream(x.device))
    return y, rstd


def rmsnorm_backward(dy: torch.Tensor, y: torch.Tensor, rstd: torch.Tensor, norm: str = "head") -> torch.Tensor:
    """dx = (dy - y mean(dy y)) rstd, the backward of :func:`rmsnorm_forward`."""
    B, H, N, dv = y.shape
    grp = _norm_group(norm, H)
    _on(y.device, y=y, dy=dy, rstd=rstd)
    dy = dy.to(y.dtype).contiguous()
    dx = torch.empty_like(y)
    _lib.call("la2_rmsnorm_backward", _ptr(dy), _ptr(y), _ptr(rstd), _ptr(dx), B, H, N, dv, grp, _code(y),
              _stream(y.device))
    return dx


def la2_forward_norm(q, k, v, decay: DecayLike, eps: float = 1e-6, norm: str = "head",
                     kv_in: Optional[torch.Tensor] = None, output_final_state: bool = False,
                     store_states: bool = False):
    """Forward with Norm(.) applied to the output (include/la2.h la2_forward_norm): fused into
    the tensor-core epilogue for bf16 per-head norms with d <= 64, dv = 64. Returns
    ``(y, rstd, kv_out, kv_blocks)``; kv_blocks (the per-block states for
    :func:`la2_backward_states`) only with ``store_states``."""
    B, H, N, d, dv = _check_qkv(q, k, v)
    if q.dtype == _F64:
        raise ValueError("Norm(.) runs on bf16 / fp32 inputs")
    grp = _norm_group(norm, H)
    dec = _decay(decay, H, q.device)
    kv_in = _state(kv_in, B, H, d, dv, q.device, "kv_in")
    kv_out = torch.empty(B, H, d, dv, device=q.device, dtype=torch.float32) if output_final_state else None
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = torch.empty_like(v)
    rstd = torch.empty(B, H // grp, N, device=q.device, dtype=torch.float32)
    blocks = (torch.empty(B, H, (N + 127) // 128, d, dv, device=q.device, dtype=torch.bfloat16)
              if store_states else None)
    _lib.call("la2_forward_norm", _ptr(q), _ptr(k), _ptr(v), _ptr(dec), _ptr(o), _ptr(kv_in), _ptr(kv_out),
              _ptr(blocks), _ptr(rstd), float(eps), grp, B, H, N, d, dv, _code(q), _stream(q.device))
    return o, rstd, kv_out, blocks


def _head_stride(t: torch.Tensor) -> Optional[int]:
    """Element stride between consecutive (b, h) rows of a [B,H,N,c] view whose rows are
    contiguous and evenly spaced (la2_forward_strided), else None."""
    B, H, N, c = t.shape
    if t.stride(3) != 1 or (N > 1 and t.stride(2) != c) or t.data_ptr() % 16:
        return None
    if B > 1 and H > 1:
        ld = t.stride(1) if t.stride(0) == H * t.stride(1) else None
    elif H > 1:
        ld = t.stride(1)
    elif B > 1:
        ld = t.stride(0)
    else:
        ld = N * c
    if ld is None or ld < N * c or ld % 8:
        return None
    return ld


def la2_backward(q, k, v, d_out, decay: DecayLike, kv_in=None, dkv_in=None, output_dkv: bool = False,
                 block: int = 0):
    """Gradients of sum(d_out * O) (tila.tiled_backward, pkg/src/tila/kernel.py:165-233).

    Returns ``(dq, dk, dv, dkv_out)``. dkv_in is the mirrored state from tokens
    after the chunk (the gradient of a downstream consumer of the final state);
    dkv_out is the mirrored state folded over the whole chunk, i.e. the gradient
    with respect to kv_in.
    """
    B, H, N, d, dv = _check_qkv(q, k, v)
    if d_out.shape != v.shape or d_out.dtype != v.dtype:
        raise ValueError(f"d_out must have shape {tuple(v.shape)} and dtype {v.dtype}")
    _on(q.device, d_out=d_out)
    if q.dtype == _F64:
        dec = _decay(decay, H, q.device, _F64)
        kv_in = _state(kv_in, B, H, d, dv, q.device, "kv_in", _F64)
        dkv_in = _state(dkv_in, B, H, d, dv, q.device, "dkv_in", _F64)
        dkv_out = torch.empty(B, H, d, dv, device=q.device, dtype=_F64) if output_dkv else None
        q, k, v, d_out = q.contiguous(), k.contiguous(), v.contiguous(), d_out.contiguous()
        dq, dk, dvv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        _lib.call("la2_backward_f64", _ptr(q), _ptr(k), _ptr(v), _ptr(d_out), _ptr(dec), _ptr(dq), _ptr(dk),
                  _ptr(dvv), _ptr(kv_in), _ptr(dkv_in), _ptr(dkv_out), B, H, N, d, dv, int(block),
                  _stream(q.device))
        return dq, dk, dvv, dkv_out
    dec = _decay(decay, H, q.device)
    kv_in = _state(kv_in, B, H, d, dv, q.device, "kv_in")
    dkv_in = _state(dkv_in, B, H, d, dv, q.device, "dkv_in")
    dkv_out = torch.empty(B, H, d, dv, device=q.device, dtype=torch.float32) if output_dkv else None
    ts = (q, k, v, d_out)
    lds = None
    if q.dtype == torch.bfloat16 and tc_shape(d, dv) and not all(t.is_contiguous() for t in ts):
        lds = [_head_stride(t) for t in ts]
        if any(x is None for x in lds):
            lds = None
    if lds is not None:  # views (chunks of a resident sequence): read in place
        dq = torch.empty(B, H, N, d, device=q.device, dtype=q.dtype)
        dk = torch.empty(B, H, N, d, device=q.device, dtype=q.dtype)
        dvv = torch.empty(B, H, N, dv, device=q.device, dtype=q.dtype)
        _lib.call("la2_backward_strided", _ptr(q), _ptr(k), _ptr(v), _ptr(d_out), _ptr(dec), _ptr(dq),
                  _ptr(dk), _ptr(dvv), _ptr(kv_in), _ptr(dkv_in), _ptr(dkv_out), B, H, N, d, dv, _code(q),
                  lds[0], lds[1], lds[2], lds[3], _stream(q.device))
        return dq, dk, dvv, dkv_out
    q, k, v, d_out = q.contiguous(), k.contiguous(), v.contiguous(), d_out.contiguous()
    dq, dk, dvv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    _lib.call("la2_backward", _ptr(q), _ptr(k), _ptr(v), _ptr(d_out), _ptr(dec), _ptr(dq), _ptr(dk),
              _ptr(dvv), _ptr(kv_in), _ptr(dkv_in), _ptr(dkv_out), B, H, N, d, dv, _code(q),
              _stream(q.device))
    return dq, dk, dvv, dkv_out


TUNE_PERSISTENT, TUNE_PREFETCH, TUNE_L2HINT, TUNE_FUSED_BWD, TUNE_CONCURRENT_BWD, TUNE_PARTITION_BWD, TUNE_PDL = 1, 2, 3, 4, 5, 6, 7


def workspace_bytes() -> int:
    """Bytes of the library's fixed per-(device, stream) workspace on the current device
    (include/la2.h la2_workspace_bytes); independent of B, H and N."""
    return int(_lib.load().la2_workspace_bytes())


def launch_log(capacity: int) -> None:
    """Start (capacity > 0) or stop (0) the library's launch log (include/la2.h
    la2_launch_log): every kernel launch is bracketed by CUDA events on its own stream."""
    _lib.call("la2_launch_log", int(capacity))


def read_launch_log(max_records: int = 65536) -> list:
    """Logged launches since the last read, in launch order: dicts with the kernel name
    (as ncu names it), grid, cluster size and event-timed ms. Waits for them."""
    buf = (_lib.LaunchRecord * max_records)()
    n = _lib.load().la2_launch_log_read(buf, max_records)
    if n < 0:
        _lib.check(n, "la2_launch_log_read")
    return [{"kernel": r.kernel.decode(), "grid": r.grid, "cluster": r.cluster, "ms": r.ms}
            for r in buf[:n]]


def set_tuning(key: int, value: int) -> None:
    """Process-wide scheduling knob of the tensor-core kernels (include/la2.h
    la2_set_tuning). Outputs do not depend on it."""
    _lib.call("la2_set_tuning", int(key), int(value))


def chunk_state(k, v, decay: DecayLike) -> torch.Tensor:
    """S = sum_s lam^(N-1-s) k_s^T v_s  (fp32 [B,H,d,dv]); sequence-parallel pass A."""
    B, H, N, d, dv = _check_qkv(k, k, v)
    k, v = k.contiguous(), v.contiguous()
    dec = _decay(decay, H, k.device)
    out = torch.empty(B, H, d, dv, device=k.device, dtype=torch.float32)
    _lib.call("la2_chunk_state", _ptr(k), _ptr(v), _ptr(dec), _ptr(out), B, H, N, d, dv, _code(k),
              _stream(k.device))
    return out


def chunk_dstate(q, d_out, decay: DecayLike) -> torch.Tensor:
    """T = sum_s lam^(s+1) q_s^T d_out_s (fp32 [B,H,d,dv]); SP backward pass A."""
    B, H, N, d, dv = _check_qkv(q, q, d_out)
    q, d_out = q.contiguous(), d_out.contiguous()
    dec = _decay(decay, H, q.device)
    out = torch.empty(B, H, d, dv, device=q.device, dtype=torch.float32)
    _lib.call("la2_chunk_dstate", _ptr(q), _ptr(d_out), _ptr(dec), _ptr(out), B, H, N, d, dv,
              _code(q), _stream(q.device))
    return out


def state_scan(states: torch.Tensor, decay: DecayLike, lens: Sequence[int],
               init: Optional[torch.Tensor] = None, reverse: bool = False) -> torch.Tensor:
    """Exclusive prefix (or suffix) combine of chunk states ``[G,B,H,d,dv]``."""
    if states.dim() != 5 or states.dtype != torch.float32 or not states.is_cuda:
        raise ValueError("states must be a CUDA float32 [G, B, H, d, dv] tensor")
    G, B, H, d, dv = states.shape
    if len(lens) != G:
        raise ValueError(f"lens must have {G} entries")
    states = states.contiguous()
    dec = _decay(decay, H, states.device)
    if init is not None:
        init = _state(init, B, H, d, dv, states.device, "init")
    out = torch.empty_like(states)
    arr = (ctypes.c_int * G)(*[int(x) for x in lens])
    _lib.call("la2_state_scan", _ptr(states), _ptr(dec), _ptr(init), _ptr(out), G, B, H, d, dv, arr,
              int(reverse), _stream(states.device))
    return out


def decode_step(q_t, k_t, v_t, decay: DecayLike, state: torch.Tensor) -> torch.Tensor:
    """One recurrent decode step, in place on ``state`` (fp32 ``[B,H,d,dv]``; float64 for
    float64 inputs).

    state <- lam*state + k_t^T v_t; returns o_t = q_t state
    (tila.inference_step, pkg/src/tila/reference.py:162-181).
    q_t, k_t: ``[B,H,d]``; v_t: ``[B,H,dv]``.
    """
    if q_t.dim() != 3 or k_t.shape != q_t.shape or v_t.dim() != 3 or v_t.shape[:2] != q_t.shape[:2]:
        raise ValueError("decode_step expects q_t, k_t [B,H,d] and v_t [B,H,dv]")
    B, H, d = q_t.shape
    dv = v_t.shape[2]
    sdt = _F64 if q_t.dtype == _F64 else torch.float32
    if tuple(state.shape) != (B, H, d, dv) or state.dtype != sdt or not state.is_contiguous():
        raise ValueError(f"state must be a contiguous {sdt} tensor of shape {(B, H, d, dv)}")
    if not (q_t.dtype == k_t.dtype == v_t.dtype):
        raise ValueError("q_t, k_t, v_t must share a dtype")
    _on(state.device, state=state, q_t=q_t, k_t=k_t, v_t=v_t)
    q_t, k_t, v_t = q_t.contiguous(), k_t.contiguous(), v_t.contiguous()
    if q_t.dtype == _F64:
        dec = _decay(decay, H, q_t.device, _F64)
        o = torch.empty_like(v_t)
        _lib.call("la2_decode_step_f64", _ptr(q_t), _ptr(k_t), _ptr(v_t), _ptr(dec), _ptr(state), _ptr(o),
                  B, H, d, dv, _stream(q_t.device))
        return o
    dec = _decay(decay, H, q_t.device)
    o = torch.empty_like(v_t)
    _lib.call("la2_decode_step", _ptr(q_t), _ptr(k_t), _ptr(v_t), _ptr(dec), _ptr(state), _ptr(o),
              B, H, d, dv, _code(q_t), _stream(q_t.device))
    return o


def decode_tokens(q, k, v, decay: DecayLike, state: torch.Tensor) -> torch.Tensor:
    """T recurrent decode steps in one launch, in place on ``state`` (fp32 ``[B,H,d,dv]``;
    float64 for float64 inputs): :func:`decode_step` folded over the T tokens -- the
    same arithmetic per token, so bit-identical to T single steps -- with the state held
    on chip across the tokens (multi-token decode: a speculative draft, a short chunk of
    a stream). q, k: ``[B,H,T,d]``; v: ``[B,H,T,dv]``; returns o ``[B,H,T,dv]``
    (tila.inference_step folded over rows, reference.py:162-181 -- tila.recurrent_forward
    continued from the state, reference.py:142-159).
    """
    if q.dim() != 4 or k.shape != q.shape or v.dim() != 4 or v.shape[:3] != q.shape[:3]:
        raise ValueError("decode_tokens expects q, k [B,H,T,d] and v [B,H,T,dv]")
    B, H, T, d = q.shape
    dv = v.shape[3]
    sdt = _F64 if q.dtype == _F64 else torch.float32
    if tuple(state.shape) != (B, H, d, dv) or state.dtype != sdt or not state.is_contiguous():
        raise ValueError(f"state must be a contiguous {sdt} tensor of shape {(B, H, d, dv)}")
    if not (q.dtype == k.dtype == v.dtype):
        raise ValueError("q, k, v must share a dtype")
    _on(state.device, state=state, q=q, k=k, v=v)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    o = torch.empty_like(v)
    if q.dtype == _F64:
        dec = _decay(decay, H, q.device, _F64)
        _lib.call("la2_decode_tokens_f64", _ptr(q), _ptr(k), _ptr(v), _ptr(dec), _ptr(state), _ptr(o),
                  B, H, T, d, dv, _stream(q.device))
        return o
    dec = _decay(decay, H, q.device)
    _lib.call("la2_decode_tokens", _ptr(q), _ptr(k), _ptr(v), _ptr(dec), _ptr(state), _ptr(o),
              B, H, T, d, dv, _code(q), _stream(q.device))
    return o


def recurrent_forward(q, k, v, decay: DecayLike, initial_state: Optional[torch.Tensor] = None):
    """Per-token recurrent forward (tila.recurrent_forward, reference.py:142-159): the
    O(N d dv) recurrence token by token from a zero (or the given) state. Returns
    ``(o, final_state)``. The tiled kernels are the throughput path; this is the
    recurrence itself, kept on the GPU for cross-checks and short streams.
    """
    B, H, N, d, dv = _check_qkv(q, k, v)
    sdt = _F64 if q.dtype == _F64 else torch.float32
    if initial_state is None:
        st = torch.zeros(B, H, d, dv, device=q.device, dtype=sdt)
    else:
        st = _state(initial_state, B, H, d, dv, q.device, "initial_state", sdt).clone()
    return decode_tokens(q, k, v, decay, st), st


# ------------------------------------------------------------------- autograd
# d = dv = 64 bf16 training: the forward stores its per-block states and the backward runs
# dQ / dK / dV as one 3-CTA cluster (la2_forward_states / la2_backward_states); False: the
# backward replays the recurrence for dQ (la2_backward)
STORED_STATES = True
# ... for sequences of at least this many tokens. Measured (B=8 H=16 d=64, one B200,
# profiles/r2b_bench_c2.json vs r2a): the triple is 1-4 % faster from N = 16K up and equal at
# 8K, but slower below, where the replay path overlaps its dQ scan with the dK/dV pair on
# partitioned SMs and the 3-CTA clusters (45 of them: 135 of 148 SMs) quantise badly.
STORED_STATES_MIN_N = 16384
class LightningAttn2Fn(torch.autograd.Function):
    """Autograd wrapper: saves q, k, v, decay (and the initial state) and
    recomputes the KV state in backward -- no per-block checkpoints, matching
    the reference's backward (pkg/src/tila/kernel.py:184-204)."""

    @staticmethod
    def forward(ctx, q, k, v, decay, initial_state, output_final_state, seq_split, norm=None, norm_eps=1e-6):
        B, H, N, d = q.shape
        g = split_factor(B, H, N, d, v.shape[3], q.dtype) if seq_split == "auto" else int(seq_split)
        ctx.stored = False
        ctx.norm = norm
        rstd = None
        stored = (STORED_STATES and N >= STORED_STATES_MIN_N and states_eligible(q, v)
                  and any(ctx.needs_input_grad[:3]))
        if g > 1:
            o, kv_out, prefix = split_forward(q, k, v, decay, g, kv_in=initial_state,
                                              output_final_state=output_final_state)
            if norm is not None:
                o, rstd = rmsnorm_forward(o, norm_eps, norm, out=o)
        elif norm is not None:
            # Norm(.) fused into the epilogue where the kernel allows it (la2_forward_norm)
            o, rstd, kv_out, prefix = la2_forward_norm(q, k, v, decay, norm_eps, norm, kv_in=initial_state,
                                                       output_final_state=output_final_state,
                                                       store_states=stored)
            ctx.stored = stored
        elif stored:
            # d = 64: keep the per-block states (half a tensor of HBM) so the backward's dQ
            # needs no replay scan and shares the dK / dV passes' reads
            o, kv_out, prefix = la2_forward_states(q, k, v, decay, kv_in=initial_state,
                                                   output_final_state=output_final_state)
            ctx.stored = True
        else:
            o, kv_out = la2_forward(q, k, v, decay, kv_in=initial_state,
                                    output_final_state=output_final_state)
            prefix = None
        ctx.g = g
        ctx.save_for_backward(q, k, v, decay, initial_state, prefix, o if norm is not None else None, rstd)
        ctx.set_materialize_grads(False)
        ctx.want_state_grad = initial_state is not None and initial_state.requires_grad
        if kv_out is None:
            return o
        return o, kv_out

    @staticmethod
    def backward(ctx, d_o, *rest):
        q, k, v, decay, initial_state, prefix, y, rstd = ctx.saved_tensors
        d_final = rest[0] if rest else None
        if d_o is None:
            d_o = torch.zeros_like(v)
        elif ctx.norm is not None:
            d_o = rmsnorm_backward(d_o, y, rstd, ctx.norm)  # through Norm(.) to the attention output
        if ctx.g > 1:
            dq, dk, dv, dkv = split_backward(q, k, v, d_o.to(q.dtype).contiguous(), decay, ctx.g, prefix,
                                             dkv_in=d_final, output_dkv=ctx.want_state_grad)
        elif ctx.stored:
            dq, dk, dv, dkv = la2_backward_states(q, k, v, d_o.to(q.dtype), decay, prefix,
                                                  dkv_in=d_final, output_dkv=ctx.want_state_grad)
        else:
            dq, dk, dv, dkv = la2_backward(q, k, v, d_o.to(q.dtype), decay, kv_in=initial_state,
                                           dkv_in=d_final, output_dkv=ctx.want_state_grad)
        return dq, dk, dv, None, dkv, None, None, None, None


def lightning_attn2(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, decay: DecayLike,
                    initial_state: Optional[torch.Tensor] = None, output_final_state: bool = False,
                    seq_split="auto", norm: Optional[str] = None, norm_eps: float = 1e-6):
    """Causal linear attention with per-head exponential decay, on the GPU.

    Args:
      q, k: ``[B, H, N, d]``; v: ``[B, H, N, dv]`` CUDA tensors, bf16, fp32 or fp64 (fp64:
        the double-precision CUDA-core path, states in fp64 too).
      decay: per-head lambda in (0, 1] -- float, sequence of H floats or a tensor.
      initial_state: optional fp32 ``[B, H, d, dv]`` state carried in.
      output_final_state: also return the fp32 final state.
      seq_split: "auto" (split long sequences into chunks when B*H is too small to
        fill the GPU, see :func:`split_factor`) or an explicit chunk count (1 = off).
      norm: None (the reference's semantics), or Norm(.) of NormAttention applied to the
        output: "head" = RMS over each head's dv features (fused into the
        tensor-core epilogue for bf16 d <= 64, dv = 64), "heads" = over all heads' features
        of a token (TransNormerLLM's SRMSNorm); bf16 / fp32 only.
    Returns ``o`` (``[B,H,N,dv]``, input dtype), or ``(o, final_state)``.
    """
    _check_qkv(q, k, v)
    sdt = _F64 if q.dtype == _F64 else torch.float32  # state / decay precision
    dec = _decay(decay, q.shape[1], q.device, sdt)
    if initial_state is not None:
        B, H, N, d = q.shape
        if tuple(initial_state.shape) != (B, H, d, v.shape[3]):
            raise ValueError(f"initial_state must have shape {(B, H, d, v.shape[3])}")
        if initial_state.dtype != sdt:
            initial_state = initial_state.to(sdt)
    if norm is not None:
        _norm_group(norm, q.shape[1])
        if q.dtype == _F64:
            raise ValueError("Norm(.) runs on bf16 / fp32 inputs")
    return LightningAttn2Fn.apply(q, k, v, dec, initial_state, bool(output_final_state), seq_split, norm,
                                  float(norm_eps))
