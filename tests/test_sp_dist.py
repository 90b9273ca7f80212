"""Sequence-parallel host logic on CPU with gloo (world sizes 2 and 4).

The local per-chunk compute is injected as fp64 NumPy ops built on the oracle
port; what is tested is paper_2401_04658_b200.sp: the chunk-state exchange
(all_gather or P2P Hillis-Steele scan), the prefix/suffix combine with
lam^L chunk factors, and the autograd wiring. Results must equal the
unsharded reference on the full sequence.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tila_port as port


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _np(t):
    return t.detach().double().numpy()


def _local_ops():
    from paper_2401_04658_b200.sp import LocalOps

    def per_bh(fn, *arrs):
        B, H = arrs[0].shape[:2]
        return [[fn(b, h) for h in range(H)] for b in range(B)]

    def chunk_state(k, v, decay):
        K, V, lam = _np(k), _np(v), decay.double().numpy()
        out = per_bh(lambda b, h: port.tiled_forward(K[b, h], K[b, h], V[b, h], lam[h], 16)[1].kv, K)
        return torch.tensor(np.asarray(out))

    def chunk_dstate(q, do, decay):
        Q, DO, lam = _np(q), _np(do), decay.double().numpy()
        n = Q.shape[2]

        def one(b, h):
            w = lam[h] ** (np.arange(n) + 1.0)
            return (Q[b, h] * w[:, None]).T @ DO[b, h]
        return torch.tensor(np.asarray(per_bh(one, Q)))

    def forward(q, k, v, decay, kv_in):
        Q, K, V, lam, S = _np(q), _np(k), _np(v), decay.double().numpy(), _np(kv_in)
        out = per_bh(lambda b, h: port.chunked_forward(Q[b, h], K[b, h], V[b, h], lam[h], 16,
                                                       port.KvState(S[b, h]))[0], Q)
        return torch.tensor(np.asarray(out))

    def backward(q, k, v, do, decay, kv_in, dkv_in):
        Q, K, V, DO = _np(q), _np(k), _np(v), _np(do)
        lam, S, T = decay.double().numpy(), _np(kv_in), _np(dkv_in)
        n = Q.shape[2]
        dq, dk, dv = np.empty_like(Q), np.empty_like(K), np.empty_like(V)
        for b in range(Q.shape[0]):
            for h in range(Q.shape[1]):
                g = port.tiled_backward(Q[b, h], K[b, h], V[b, h], DO[b, h], lam[h], 16)
                read = lam[h] ** (np.arange(n) + 1.0)
                write = lam[h] ** (n - 1.0 - np.arange(n))
                dq[b, h] = g.dq + (DO[b, h] * read[:, None]) @ S[b, h].T
                dk[b, h] = g.dk + (V[b, h] * write[:, None]) @ T[b, h].T
                dv[b, h] = g.dv + (K[b, h] * write[:, None]) @ T[b, h]
        return torch.tensor(dq), torch.tensor(dk), torch.tensor(dv)

    return LocalOps(chunk_state, chunk_dstate, forward, backward)


def _worker(rank, world, port_no, mode, lens, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2401_04658_b200.sp import sp_lightning_attn2

        B, H, d, dv = 1, 3, 4, 5
        N = sum(lens)
        decay = torch.tensor([0.875, 1 - 2 ** -10, 1.0], dtype=torch.float64)  # exact in fp32
        q, k, v, do = (torch.tensor(port.random_matrix(B * H * N, c, 300 + i).reshape(B, H, N, c))
                       for i, c in enumerate((d, d, dv, dv)))
        a = sum(lens[:rank])
        sl = slice(a, a + lens[rank])
        ql, kl, vl = (t[:, :, sl].clone().requires_grad_() for t in (q, k, v))
        o = sp_lightning_attn2(ql, kl, vl, decay, mode=mode, local_ops=_local_ops())
        o.backward(do[:, :, sl])
        result_q.put((rank, _np(o), _np(ql.grad), _np(kl.grad), _np(vl.grad)))
    except Exception:  # report instead of hanging the parent
        import traceback

        result_q.put((rank, "error", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["allgather", "p2p"])
@pytest.mark.parametrize("lens", [[40, 24], [17, 30, 9, 44]])
def test_sp_matches_unsharded(mode, lens):
    world = len(lens)
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, mode, lens, q_)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        r, *arrs = q_.get(timeout=240)
        assert not (len(arrs) == 2 and arrs[0] == "error"), arrs[1]
        results[r] = arrs
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    B, H, d, dv = 1, 3, 4, 5
    N = sum(lens)
    decay = [0.875, 1 - 2 ** -10, 1.0]
    q, k, v, do = (port.random_matrix(B * H * N, c, 300 + i).reshape(B, H, N, c)
                   for i, c in enumerate((d, d, dv, dv)))
    ro = port.bhnd_oracle_forward(q, k, v, decay)
    rq, rk, rv = port.bhnd_oracle_backward(q, k, v, do, decay)
    cat = [np.concatenate([results[r][i] for r in range(world)], axis=2) for i in range(4)]
    for got, ref in zip(cat, (ro, rq, rk, rv)):
        assert port.rel_err(got, ref) <= 1e-10
