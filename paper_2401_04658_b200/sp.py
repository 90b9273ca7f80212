"""Sequence parallelism for one long sequence: each rank owns a contiguous chunk.

Exact three-phase scheme. Forward:
  A. S_g = chunk-local final state of rank g's chunk from zero
     (= tila.chunked_forward's KvState.kv from a fresh state, pkg/src/tila/kernel.py:142-162);
  B. exchange + exclusive prefix  KV_in(g) = sum_{g'<g} (prod_{g'<j<g} lam^L_j) S_g'
     -- the block fold KV <- lam^r KV + dKV of pkg/src/tila/kernel.py:111-115 applied per chunk;
  C. the local pass with kv_in = KV_in(g).
Backward mirrors it with the reverse-sweep state of tiled_backward
(pkg/src/tila/kernel.py:207-231): T_g from zero, exclusive SUFFIX combine into
dKV_in(g), then the local backward with (KV_in(g), dKV_in(g)).

The only collective is the [B,H,d,dv] fp32 state exchange, one per direction:
``mode="allgather"`` (one all_gather, local combine) or ``mode="p2p"``
(Hillis-Steele scan, ceil(log2 G) rounds of send/recv plus one shift).
The local compute is injected (``LocalOps``): the CUDA kernels in production,
any torch-tensor implementation in CPU multi-process tests.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


@dataclass
class LocalOps:
    chunk_state: Callable    # (k, v, decay) -> S
    chunk_dstate: Callable   # (q, do, decay) -> T
    forward: Callable        # (q, k, v, decay, kv_in) -> o
    backward: Callable       # (q, k, v, do, decay, kv_in, dkv_in) -> (dq, dk, dv)


def cuda_ops(seq_split="auto") -> LocalOps:
    """The CUDA kernels as the local compute of one rank, composed with the intra-GPU
    sequence split (ops.split_factor): with few heads a rank's chunk alone would fill a
    fraction of the SMs (C5: 16 heads x 2 value slices = 32 CTAs), so each rank cuts its
    chunk into g sub-chunks and runs the same three phases inside the GPU:

      pass A   sub-chunk states S_j (one chunk_state launch over B*H*g units), combined
               locally into the rank's chunk state S = lam^(L/g) P_(g-1) + S_(g-1), where
               P = exclusive prefix of the S_j from zero (la2_state_scan);
      exchange S across ranks -> KV_in (the caller, exclusive_scan);
      pass B   sub-chunk carries = exclusive prefix of the S_j seeded with KV_in
               (la2_state_scan with init), then one forward over the B*H*g units.

    The backward mirrors it with the reverse-sweep states (chunk_dstate, suffix scans).
    Exact algebra (the fold of pkg/src/tila/kernel.py:111-115 per sub-chunk); returns a
    fresh object per autograd call (it keeps the sub-chunk states of that call).
    """
    from . import ops

    st: dict = {}

    def factor(B, H, L, d, dv, dtype):
        g = ops.split_factor(B, H, L, d, dv, dtype) if seq_split == "auto" else int(seq_split)
        return g if g > 1 and L % g == 0 else 1

    def chunk_state(k, v, dec):
        B, H, L, d = k.shape
        dv = v.shape[3]
        g = st["g"] = factor(B, H, L, d, dv, k.dtype)
        if g == 1:
            return ops.chunk_state(k, v, dec)
        dec_g = ops.decay_repeat(dec, g)
        s = ops.chunk_state(ops._chunked(k.contiguous(), g), ops._chunked(v.contiguous(), g), dec_g)
        s5 = st["s5"] = ops._to_chunk_major(s, B, H, g)
        pre = ops.state_scan(s5, dec, [L // g] * g)
        return _decay_pow(dec, torch.tensor(L // g)) * pre[-1] + s5[-1]

    def forward(q, k, v, dec, kv_in):
        B, H, L, d = q.shape
        g = st.get("g", 1)
        if g == 1:
            return ops.la2_forward(q, k, v, dec, kv_in=kv_in)[0]
        prefix = ops._from_chunk_major(ops.state_scan(st["s5"], dec, [L // g] * g, init=kv_in), B, H, g)
        q4, k4, v4 = (ops._chunked(t.contiguous(), g) for t in (q, k, v))
        o4, _ = ops.la2_forward(q4, k4, v4, ops.decay_repeat(dec, g), kv_in=prefix)
        return o4.view(B, H, L, v.shape[3])

    def chunk_dstate(q, do, dec):
        B, H, L, d = q.shape
        dv = do.shape[3]
        g = st["g"] = factor(B, H, L, d, dv, q.dtype)
        if g == 1:
            return ops.chunk_dstate(q, do, dec)
        t = ops.chunk_dstate(ops._chunked(q.contiguous(), g), ops._chunked(do.contiguous(), g),
                             ops.decay_repeat(dec, g))
        t5 = st["t5"] = ops._to_chunk_major(t, B, H, g)
        suf = ops.state_scan(t5, dec, [L // g] * g, reverse=True)
        return _decay_pow(dec, torch.tensor(L // g)) * suf[0] + t5[0]

    def backward(q, k, v, do, dec, kv_in, dkv_in):
        B, H, L, d = q.shape
        dv = v.shape[3]
        g = st.get("g", 1)
        if g == 1:
            return ops.la2_backward(q, k, v, do, dec, kv_in=kv_in, dkv_in=dkv_in)[:3]
        if "s5" not in st:  # backward without this object's forward: recompute pass A
            chunk_state(k, v, dec)
        lens = [L // g] * g
        prefix = ops._from_chunk_major(ops.state_scan(st["s5"], dec, lens, init=kv_in), B, H, g)
        suffix = ops._from_chunk_major(ops.state_scan(st["t5"], dec, lens, init=dkv_in, reverse=True),
                                       B, H, g)
        q4, k4, v4, do4 = (ops._chunked(t.contiguous(), g) for t in (q, k, v, do))
        dq, dk, dvv, _ = ops.la2_backward(q4, k4, v4, do4, ops.decay_repeat(dec, g), kv_in=prefix,
                                          dkv_in=suffix)
        return dq.view(B, H, L, d), dk.view(B, H, L, d), dvv.view(B, H, L, dv)

    ops_ = LocalOps(chunk_state=chunk_state, chunk_dstate=chunk_dstate, forward=forward,
                    backward=backward)
    ops_.split = st  # introspection (tests, bench): st["g"] is the sub-chunk count used
    return ops_


def _decay_pow(decay: torch.Tensor, length: torch.Tensor, dtype=torch.float32) -> torch.Tensor:
    """lam_h ** L as [1, H, 1, 1] in the state dtype (computed in fp64, underflow -> 0)."""
    f = torch.pow(decay.double(), length.double())
    f = torch.where(f < torch.finfo(dtype).tiny, torch.zeros_like(f), f)
    return f.to(dtype).reshape(1, -1, 1, 1)


def exclusive_scan(state: torch.Tensor, decay: torch.Tensor, length: int, group=None,
                   reverse: bool = False, mode: str = "allgather") -> torch.Tensor:
    """Exclusive prefix (reverse: suffix) combine of per-rank chunk states.

    state: this rank's [B,H,d,dv] fp32 chunk state; decay: [H]; length: this
    rank's chunk length. Returns the state carried into this rank's chunk.
    """
    G = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = state.device
    if state.is_cuda and dist.get_backend(group) == "gloo":
        # gloo moves host memory only: stage the (small, [B,H,d,dv]) state through the host
        out = exclusive_scan(state.cpu(), decay.cpu(), length, group, reverse, mode)
        return out.to(dev)
    decay = decay.to(dev)
    lens = torch.tensor([length], dtype=torch.int64, device=dev)
    if G == 1:
        return torch.zeros_like(state)
    if mode == "allgather":
        buf = [torch.empty_like(state) for _ in range(G)]
        dist.all_gather(buf, state.contiguous(), group=group)
        all_lens = [torch.empty_like(lens) for _ in range(G)]
        dist.all_gather(all_lens, lens, group=group)
        order = range(G - 1, rank, -1) if reverse else range(rank)
        acc = torch.zeros_like(state)
        for g in order:
            acc = _decay_pow(decay, all_lens[g][0], state.dtype) * acc + buf[g]
        return acc
    if mode == "p2p":
        return _p2p_scan(state, decay, lens, group, reverse, G, rank)
    raise ValueError(f"unknown exchange mode {mode!r} (expected 'allgather' or 'p2p')")


def _p2p_scan(state, decay, lens, group, reverse, G, rank):
    """Hillis-Steele inclusive scan with (A, F) o (A', F') = (F' A + A', F F'),
    then a one-step shift to make it exclusive. Virtual order is reversed for
    the suffix (backward) scan."""
    vr = G - 1 - rank if reverse else rank
    to_rank = (lambda v: G - 1 - v) if reverse else (lambda v: v)
    glob = lambda r: dist.get_global_rank(group, r) if group is not None else r  # noqa: E731
    A = state.contiguous().clone()
    F = _decay_pow(decay, lens[0], state.dtype).contiguous().clone()
    off = 1
    while off < G:
        ops_ = []
        recv_A = torch.empty_like(A)
        recv_F = torch.empty_like(F)
        if vr + off < G:
            ops_ += [dist.P2POp(dist.isend, A, glob(to_rank(vr + off)), group),
                     dist.P2POp(dist.isend, F, glob(to_rank(vr + off)), group)]
        if vr - off >= 0:
            ops_ += [dist.P2POp(dist.irecv, recv_A, glob(to_rank(vr - off)), group),
                     dist.P2POp(dist.irecv, recv_F, glob(to_rank(vr - off)), group)]
        if ops_:
            for w in dist.batch_isend_irecv(ops_):
                w.wait()
        if vr - off >= 0:
            A = F * recv_A + A
            F = recv_F * F
        off *= 2
    # shift: exclusive(v) = inclusive(v - 1)
    out = torch.zeros_like(A)
    ops_ = []
    if vr + 1 < G:
        ops_.append(dist.P2POp(dist.isend, A, glob(to_rank(vr + 1)), group))
    if vr - 1 >= 0:
        ops_.append(dist.P2POp(dist.irecv, out, glob(to_rank(vr - 1)), group))
    if ops_:
        for w in dist.batch_isend_irecv(ops_):
            w.wait()
    return out


class SPLightningAttn2Fn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, decay, group, mode, local_ops):
        n = q.shape[2]
        s = local_ops.chunk_state(k, v, decay)
        kv_in = exclusive_scan(s, decay, n, group, reverse=False, mode=mode)
        o = local_ops.forward(q, k, v, decay, kv_in)
        ctx.save_for_backward(q, k, v, decay, kv_in)
        ctx.group, ctx.mode, ctx.local_ops = group, mode, local_ops
        return o

    @staticmethod
    def backward(ctx, d_o):
        q, k, v, decay, kv_in = ctx.saved_tensors
        d_o = d_o.contiguous().to(q.dtype)
        t = ctx.local_ops.chunk_dstate(q, d_o, decay)
        dkv_in = exclusive_scan(t, decay, q.shape[2], ctx.group, reverse=True, mode=ctx.mode)
        dq, dk, dv = ctx.local_ops.backward(q, k, v, d_o, decay, kv_in, dkv_in)
        return dq, dk, dv, None, None, None, None


def sp_lightning_attn2(q, k, v, decay, group=None, mode: str = "allgather",
                       local_ops: Optional[LocalOps] = None, seq_split="auto"):
    """Sequence-parallel lightning_attn2 over ``group``.

    Each rank passes its contiguous chunk ``[B, H, N_g, d]`` of one long
    sequence (rank order = sequence order); the result is this rank's chunk of
    the output of the unsharded op. ``decay``: [H] tensor on the local device.
    ``seq_split``: sub-chunks per rank for the intra-GPU split ("auto" =
    ops.split_factor of the rank's chunk, 1 = off); see :func:`cuda_ops`.
    """
    ops_ = local_ops if local_ops is not None else cuda_ops(seq_split)
    if not isinstance(decay, torch.Tensor):
        decay = torch.tensor(decay, dtype=torch.float32, device=q.device)
    return SPLightningAttn2Fn.apply(q, k, v, decay.float().contiguous(), group, mode, ops_)
