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


def cuda_ops() -> LocalOps:
    from . import ops

    return LocalOps(
        chunk_state=ops.chunk_state,
        chunk_dstate=ops.chunk_dstate,
        forward=lambda q, k, v, dec, kv_in: ops.la2_forward(q, k, v, dec, kv_in=kv_in)[0],
        backward=lambda q, k, v, do, dec, kv_in, dkv_in: ops.la2_backward(
            q, k, v, do, dec, kv_in=kv_in, dkv_in=dkv_in)[:3],
    )


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
                       local_ops: Optional[LocalOps] = None):
    """Sequence-parallel lightning_attn2 over ``group``.

    Each rank passes its contiguous chunk ``[B, H, N_g, d]`` of one long
    sequence (rank order = sequence order); the result is this rank's chunk of
    the output of the unsharded op. ``decay``: [H] tensor on the local device.
    """
    ops_ = local_ops if local_ops is not None else cuda_ops()
    if not isinstance(decay, torch.Tensor):
        decay = torch.tensor(decay, dtype=torch.float32, device=q.device)
    return SPLightningAttn2Fn.apply(q, k, v, decay.float().contiguous(), group, mode, ops_)
