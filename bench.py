#!/usr/bin/env python
"""Benchmark of the Lightning-2 hot path (fwd+bwd) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the metric's configuration): the
TransNormerLLM-400M attention shape B=8, H=16, d=dv=64, bf16, one step = one
forward + backward pass of all heads at seq_len N (default 65536, the top of
the 1K-64K sweep; every input tensor is 1 GiB, far larger than the 126 MB L2,
so no flush is needed between steps). The full 1K-64K sweep is measured in
the same run and reported under "sweep". Inputs are synthetic
(torch.rand * 2 - 1), decay lam_h = exp(-2^(-8(h+1)/H)).

Multi-GPU (torchrun): each rank runs its own B=8 batch (batch x head sharding,
no collective on the data path, "scaling": "weak"); time = max over ranks.

--impl reference: the reference's own CPU implementation (tila.tiled_forward /
tiled_backward from oracle/_ref/tila, the unmodified package staged by build(); the
oracle port of pkg/src/tila/kernel.py if it is absent), numpy/OpenBLAS on all host
cores of rank 0, over a bounded sample of the same workload, extrapolated to the same
metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fwd+bwd tokens/s (B=8,H=16,d=64 bf16, 1K-64K sweep)"
UNIT = "tokens/s"


def alibi_decay(H: int) -> list[float]:
    return [math.exp(-(2.0 ** (-8.0 * (h + 1) / H))) for h in range(H)]


def canonical_flops(N, d, dv):
    """F_fwd = N[2*64(d+dv) + 4 d dv], F_bwd = N[2*64(3d+2dv) + 10 d dv]."""
    return N * (2 * 64 * (d + dv) + 4 * d * dv), N * (2 * 64 * (3 * d + 2 * dv) + 10 * d * dv)


def canonical_bytes(N, d, dv, e=2):
    """Compulsory HBM bytes: fwd e*N*(2d+2dv), bwd e*N*(4d+3dv) per (b, h)."""
    return e * N * (2 * d + 2 * dv), e * N * (4 * d + 3 * dv)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled every 20 ms through NVML while the
    timed region runs (falls back to nvidia-smi if pynvml is unavailable)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, reasons_mask, util)
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons

            def power_violation_ns():
                try:
                    return nv.nvmlDeviceGetViolationStatus(h, nv.NVML_PERF_POLICY_POWER).violationTime
                except Exception:
                    return None

            self._viol0 = power_violation_ns()
            self._viol_fn = power_violation_ns
            while not self._stop.is_set():
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), get_reasons(h),
                                     nv.nvmlDeviceGetUtilizationRates(h).gpu))
                self._stop.wait(0.02)
        except Exception as exc:  # pragma: no cover - reported in the JSON
            self.error = repr(exc)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        busy = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = sorted({name for s in busy for bit, name in self.REASONS.items() if s[1] & bit})
        # NVML's power-violation counter catches SW power capping shorter than the 20 ms
        # sampling period (sustained HBM-heavy load trips it while SM clocks read max)
        cap_ms = None
        v0, fn = getattr(self, "_viol0", None), getattr(self, "_viol_fn", None)
        if v0 is not None and fn is not None:
            v1 = fn()
            if v1 is not None:
                cap_ms = (v1 - v0) / 1e6
                if cap_ms > 0 and "sw_power_cap" not in reasons:
                    reasons = sorted(reasons + ["sw_power_cap"])
        return {"sm_mhz": statistics.median([s[0] for s in busy]) if busy else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "power_cap_ms": cap_ms, "source": "nvml"}


# ------------------------------------------------------------------ CPU side
REF_PKG = ROOT / "oracle" / "_ref"  # the reference package itself, staged by build()


def _reference_impl():
    """The reference's own tiled_forward / tiled_backward (oracle/_ref/tila, staged by
    build() from /root/reference) when present, else the oracle port's restatement."""
    if (REF_PKG / "tila" / "kernel.py").exists():
        if str(REF_PKG) not in sys.path:
            sys.path.insert(0, str(REF_PKG))
        import tila

        return tila, "reference"
    from oracle import tila_port as port

    return port, "port"


def _cpu_head_task(args):
    n, d, seed, lam = args
    import numpy as np

    impl, _ = _reference_impl()
    rng = np.random.default_rng(seed)
    q, k, v, do = (rng.uniform(-1, 1, (n, d)).astype(np.float32) for _ in range(4))
    t0 = time.perf_counter()
    impl.tiled_forward(q, k, v, lam, 64)
    impl.tiled_backward(q, k, v, do, lam, 64)
    return time.perf_counter() - t0


def cpu_reference(n: int, d: int, heads_total: int, tokens_per_step: int, sample_heads: int,
                  reps: int = 1):
    """Time the reference algorithm (oracle port, fp32, block 64) per head on
    all host cores; extrapolate to the full B*H workload."""
    import concurrent.futures as cf
    import multiprocessing as mp

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    cores = len(os.sched_getaffinity(0))
    sample_heads = max(sample_heads, cores)
    decay = alibi_decay(16)
    tasks = [(n, d, 1000 + i, decay[i % 16]) for i in range(sample_heads)]
    ctx = mp.get_context("spawn")
    with cf.ProcessPoolExecutor(max_workers=cores, mp_context=ctx) as ex:
        list(ex.map(_cpu_head_task, tasks[:cores]))  # warm-up
        walls = []
        for _ in range(reps):
            t0 = time.perf_counter()
            list(ex.map(_cpu_head_task, tasks))
            walls.append(time.perf_counter() - t0)
    wall = statistics.median(walls)
    t_full = wall * heads_total / sample_heads
    kind = _reference_impl()[1]
    return {"value": tokens_per_step / t_full, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{sample_heads} heads x N={n} d={d} fp32 fwd+bwd "
                      f"({'the reference tila.tiled_forward/tiled_backward' if kind == 'reference' else 'oracle port of the tila block loop'}, block=64), "
                      f"{cores} processes, median of {reps}; extrapolated x{heads_total / sample_heads:.1f} "
                      f"to B*H={heads_total}",
            "sample_wall_s": wall}


# ------------------------------------------------------------------ GPU side
def c5_phases(q, k, v, do, dec, world, timed_phase):
    """C5 per-rank time split: pass A (chunk states), the exchange (state
    scan across ranks -- NCCL -- or across the intra-GPU chunks), pass B (the F passes
    with the carried states), forward and backward, each timed alone on the device."""
    from paper_2401_04658_b200 import ops
    from paper_2401_04658_b200.sp import exclusive_scan
    B, H, L, D = q.shape
    res = {}
    if world > 1:
        from paper_2401_04658_b200.sp import cuda_ops
        mode = os.environ.get("LA2_SP_MODE", "allgather")
        local = cuda_ops("auto")  # the rank's chunk, split into sub-chunks inside the GPU
        s = local.chunk_state(k, v, dec)
        kv_in = exclusive_scan(s, dec, L, None, reverse=False, mode=mode)
        t = local.chunk_dstate(q, do, dec)
        dkv_in = exclusive_scan(t, dec, L, None, reverse=True, mode=mode)
        res["sub_chunks_per_rank"] = local.split.get("g", 1)
        res["fwd_pass_a"] = timed_phase(lambda: local.chunk_state(k, v, dec))
        res["fwd_exchange"] = timed_phase(lambda: exclusive_scan(s, dec, L, None, mode=mode))
        res["fwd_pass_b"] = timed_phase(lambda: local.forward(q, k, v, dec, kv_in))
        res["bwd_pass_a"] = timed_phase(lambda: local.chunk_dstate(q, do, dec))
        res["bwd_exchange"] = timed_phase(lambda: exclusive_scan(t, dec, L, None, reverse=True, mode=mode))
        res["bwd_pass_b"] = timed_phase(lambda: local.backward(q, k, v, do, dec, kv_in, dkv_in))
        res["exchange_bytes_per_direction"] = 2 * world * H * D * D * 4
        return res
    g = ops.split_factor(B, H, L, D, D, q.dtype)
    if g == 1:
        return {"note": "no split at this shape"}
    dec_g = dec.repeat_interleave(g)
    q4, k4, v4, do4 = (ops._chunked(x.contiguous(), g) for x in (q, k, v, do))
    lens = [L // g] * g
    s = ops.chunk_state(k4, v4, dec_g)
    s5 = ops._to_chunk_major(s, B, H, g)
    prefix = ops._from_chunk_major(ops.state_scan(s5, dec, lens), B, H, g)
    t = ops.chunk_dstate(q4, do4, dec_g)
    t5 = ops._to_chunk_major(t, B, H, g)
    suffix = ops._from_chunk_major(ops.state_scan(t5, dec, lens, reverse=True), B, H, g)
    res["chunks"] = g
    res["fwd_pass_a"] = timed_phase(lambda: ops.chunk_state(k4, v4, dec_g))
    res["fwd_exchange"] = timed_phase(lambda: ops.state_scan(s5, dec, lens))
    res["fwd_pass_b"] = timed_phase(lambda: ops.la2_forward(q4, k4, v4, dec_g, kv_in=prefix))
    res["bwd_pass_a"] = timed_phase(lambda: ops.chunk_dstate(q4, do4, dec_g))
    res["bwd_exchange"] = timed_phase(lambda: ops.state_scan(t5, dec, lens, reverse=True))
    res["bwd_pass_b"] = timed_phase(lambda: ops.la2_backward(q4, k4, v4, do4, dec_g, kv_in=prefix,
                                                             dkv_in=suffix))
    return res


def _oracle_head_task(args):
    """fp64 tiled forward + backward of one head (the pinned oracle port, block 64)."""
    q, k, v, do, lam = args
    from oracle import tila_port as port

    o, _ = port.tiled_forward(q, k, v, lam, 64)
    g = port.tiled_backward(q, k, v, do, lam, 64)
    return o, g.dq, g.dk, g.dv


def parity_spot_check(heads, tol=1e-2):
    """heads: list of (label, lam, q, k, v, do, o, dq, dk, dv) numpy arrays of one head, the
    inputs as the GPU saw them (bf16 values) and the GPU outputs. Compares against the fp64
    oracle with the reference's metric (verify.py:50-75) in a process pool."""
    import concurrent.futures as cf
    import multiprocessing as mp

    from oracle import tila_port as port

    tasks = [(h[2], h[3], h[4], h[5], h[1]) for h in heads]
    with cf.ProcessPoolExecutor(max_workers=len(tasks), mp_context=mp.get_context("spawn")) as ex:
        refs = list(ex.map(_oracle_head_task, tasks))
    rows = []
    for h, ref in zip(heads, refs):
        errs = {n: port.rel_err(got, r) for n, got, r in zip(("o", "dq", "dk", "dv"), h[6:10], ref)}
        rows.append({"head": h[0], "lam": h[1], "rel_err": errs})
    worst = max(max(r["rel_err"].values()) for r in rows)
    return {"oracle": "oracle/tila_port.py tiled fp64 (block 64) on the same bf16 inputs",
            "metric": "max|gpu-ref|/max|ref| (verify.py:50-75)", "tol": tol, "heads": rows,
            "max_rel_err": worst, "pass": bool(worst <= tol)}


def launch_roles(recs, roles):
    """Group a launch log by role: recs is the log of `steps` calls whose per-call launch
    pattern is roles (a list of role names, one per launch of one call)."""
    out = {}
    if not recs or len(recs) % len(roles):
        return out
    for i, r in enumerate(recs):
        role = roles[i % len(roles)]
        e = out.setdefault(role, {"kernel": r["kernel"], "grid": r["grid"], "cluster": r["cluster"],
                                  "ms": []})
        e["ms"].append(r["ms"])
    for e in out.values():
        e["ms"] = statistics.median(e["ms"])
    return out


def load_ncu_bytes(d: int):
    """DRAM bytes per (token, head) of each launch of one fwd+bwd step (d = 64: forward F
    with stored states, dQ/dK/dV triple; or forward F, dQ F, dK/dV pair) from the committed
    ncu --set full capture (profiles/ncu_summary.json)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        j = json.loads(p.read_text())
        key = f"full_d{d}"
        th = j["token_heads"][key]
        ls = j["launches"][key]
        roles = {2: ("forward", "backward"), 3: ("forward", "dq", "dkdv")}.get(len(ls))
        if roles is None:
            return None
        return {role: (x["dram_read_bytes"] + x["dram_write_bytes"]) / th for role, x in zip(roles, ls)}
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--dim", type=int, default=64)
    ap.add_argument("--seq-len", type=int, default=65536)
    ap.add_argument("--soak-s", type=float, default=1.0,
                    help="seconds of back-to-back steps before the timed (sustained) steps")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--cpu-sample-heads", type=int, default=48)
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="c2 (default) = the headline BASELINE configs[1]; c1/c3/c4/c5 = the other configs")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload != "c2" and args.impl == "ours":
        return extra_workload(args, world, rank, local_rank)
    B, H, N, D = args.batch, args.heads, args.seq_len, args.dim
    config = {"workload": "TransNormerLLM-400M attention (BASELINE configs[1]) fwd+bwd" if D == 64 else
              f"BASELINE configs[1] shape at head dim {D} (split-d variant)" if D == 256 else
              f"BASELINE configs[1] shape at head dim {D}",
              "batch_per_gpu": B, "global_batch": B * world, "heads": H, "head_dim": D,
              "seq_len": N, "decay": "alibi-style exp(-2^(-8(h+1)/H))",
              "parallelism": f"bxh-shard x{world}" if world > 1 else "single",
              "l2": "inputs (1 GiB/tensor at N=64K) larger than L2; no flush",
              "timing": f"sustained: {args.soak_s:g} s of back-to-back steps, then the K timed steps"}

    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_reference(N, D, B * H * world, B * N * world, args.cpu_sample_heads, reps=max(1, min(3, args.steps)))
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "fp32", "data": "synthetic", "config": config,
                          "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                          "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist

    import paper_2401_04658_b200 as la2
    from paper_2401_04658_b200 import ops

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lams = alibi_decay(H)
    decay = la2.decay_tensor(lams, H, dev)

    def make(n, seed):
        g = torch.Generator(device=dev).manual_seed(seed + 1000 * rank)
        return [(torch.rand(B, H, n, D, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
                for _ in range(4)]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # what the autograd entry point runs at a shape (ops.LightningAttn2Fn's policy)
    use_stored = lambda n: ops.STORED_STATES and D == 64 and n >= ops.STORED_STATES_MIN_N  # noqa: E731
    stored = use_stored(N)

    def step(q, k, v, do):
        # the device work of one lightning_attn2 training step (LightningAttn2Fn): d = 64
        # stores the per-block states and runs the dQ/dK/dV triple; otherwise replay
        if use_stored(q.shape[2]):
            _, _, blocks = ops.la2_forward_states(q, k, v, decay)
            ops.la2_backward_states(q, k, v, do, decay, blocks)
        else:
            la2.la2_forward(q, k, v, decay)
            la2.la2_backward(q, k, v, do, decay)

    def run_timed(fn, steps):
        """Device time per call of `steps` back-to-back calls (events on torch's current
        stream, which is the stream the library launches on)."""
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    def time_steps(fn, steps, warmup, soak_s=0.0):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        soak = None
        if soak_s > 0:
            # bring the board to its steady state (power limit) before the timed steps
            probe = run_timed(fn, 2)
            n_soak = max(4, int(math.ceil(soak_s * 1e3 / max(probe, 1e-3))))
            soak = {"steps": n_soak, "ms_per_step": run_timed(fn, n_soak)}
            soak["window_s"] = soak["ms_per_step"] * n_soak / 1e3
        barrier()
        torch.cuda.synchronize()
        ms = run_timed(fn, steps) if steps > 0 else 0.0
        barrier()
        return max_over_ranks(ms), soak

    hbm_peak, tc_peak, peak_src = load_peaks()
    ff, fb = canonical_flops(N, D, D)
    bf, bb = canonical_bytes(N, D, D)

    # ---------------- burst: K steps on a rested GPU (reported beside the headline)
    q, k, v, do = make(N, 0)
    ms_burst, _ = time_steps(lambda: step(q, k, v, do), args.steps, max(3, args.warmup))

    # ---------------- per-launch times (launch log: events on the launching stream)
    # in the sustained regime, like the headline
    time_steps(lambda: step(q, k, v, do), 0, 0, soak_s=args.soak_s)
    ops.launch_log(16 * max(3, args.steps) + 8)
    blocks = None
    for _ in range(max(3, args.steps)):
        if stored:
            _, _, blocks = ops.la2_forward_states(q, k, v, decay)
        else:
            la2.la2_forward(q, k, v, decay)
    fwd_log = ops.read_launch_log()
    for _ in range(max(3, args.steps)):
        if stored:
            ops.la2_backward_states(q, k, v, do, decay, blocks)
        else:
            la2.la2_backward(q, k, v, do, decay)
    bwd_log = ops.read_launch_log()
    ops.launch_log(0)
    del blocks
    n_f = max(3, args.steps)
    per_call_f, per_call_b = len(fwd_log) // n_f, len(bwd_log) // n_f
    if per_call_f == 1 and per_call_b == 1:  # d = 64 stored states: forward F | dQ/dK/dV triple
        roles = launch_roles(fwd_log, ["forward"])
        roles.update(launch_roles(bwd_log, ["backward"]))
    elif per_call_f == 1 and per_call_b == 2:  # d = 64 replay: forward F | dQ F, dK/dV pair
        roles = launch_roles(fwd_log, ["forward"])
        roles.update(launch_roles(bwd_log, ["dq", "dkdv"]))
    else:  # other shapes (split-d, separate dK / dV passes): one entry per direction
        roles = {}
        for name, log, per in (("forward", fwd_log, per_call_f), ("backward", bwd_log, per_call_b)):
            r = launch_roles(log, [f"{name}{i}" for i in range(per)])
            if r:
                roles[name] = {"kernel": " + ".join(sorted({x["kernel"] for x in r.values()})),
                               "grid": max(x["grid"] for x in r.values()),
                               "cluster": max(x["cluster"] for x in r.values()),
                               "ms": sum(x["ms"] for x in r.values()), "launches_per_call": per}
    launches_per_step = per_call_f + per_call_b

    # ---------------- headline: sustained (soak, then exactly K timed steps)
    clocks = ClockSampler(local_rank).start()
    ms, soak = time_steps(lambda: step(q, k, v, do), args.steps, max(3, args.warmup), soak_s=args.soak_s)
    clk = clocks.stop()
    tokens_step = B * N * world
    value = tokens_step / (ms / 1e3)
    tflops = (ff + fb) * B * H * world / (ms / 1e3) / 1e12
    t_roof = max((ff + fb) * B * H / (tc_peak * 1e12), (bf + bb) * B * H / (hbm_peak * 1e9)) * 1e3

    # ---------------- roofline per launch; the dominant kernel is the one with the largest share
    e = 2
    alg = {"forward": B * H * N * e * (2 * D + 2 * D),   # read q, k, v; write o
           "dq": B * H * N * e * (2 * D + 2 * D),        # read dO, V, K; write dQ
           "dkdv": B * H * N * e * (3 * D + 3 * D),      # read K, Q, dO, V; write dK, dV
           "backward": bb * B * H}                        # SURVEY 8d compulsory backward bytes
    ncu_bytes = load_ncu_bytes(D)
    launches = []
    for role, r in roles.items():
        a_bytes = alg.get(role)
        ent = {"role": role, "kernel": r["kernel"], "grid": r["grid"], "cluster": r["cluster"],
               "launch_ms": r["ms"]}
        if "launches_per_call" in r:
            ent["launches_per_call"] = r["launches_per_call"]
        if a_bytes:
            ach = a_bytes / (r["ms"] / 1e3) / 1e9
            ent.update({"algorithmic_bytes": a_bytes, "achieved_gbs": ach, "frac": ach / hbm_peak,
                        "traffic": (ncu_bytes[role] * B * H * N) if ncu_bytes and role in ncu_bytes
                        else None})
        launches.append(ent)
    sum_launch = sum(x["launch_ms"] for x in launches) or 1.0
    for x in launches:
        x["share_of_step"] = x["launch_ms"] / sum_launch
    dom = max(launches, key=lambda x: x["launch_ms"]) if launches else None
    step_alg = (bf + bb) * B * H
    step_traffic = sum(ncu_bytes.values()) * B * H * N if ncu_bytes else None
    roofline = {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak, "peak_source": peak_src,
                "kernel": dom and dom["kernel"], "role": dom and dom["role"],
                "achieved": dom and dom.get("achieved_gbs"), "frac": dom and dom.get("frac"),
                "algorithmic_bytes_per_launch": dom and dom.get("algorithmic_bytes"),
                "traffic": dom and dom.get("traffic"), "launch_ms": dom and dom["launch_ms"],
                "launches": launches,
                "step": {"t_roof_ms": t_roof, "t_ms": ms, "frac_of_roof": t_roof / ms,
                         "tflops": tflops, "frac_of_bf16_peak": tflops / tc_peak,
                         "algorithmic_bytes": step_alg, "dram_bytes_ncu": step_traffic,
                         "traffic_ratio": (step_traffic / step_alg) if step_traffic else None,
                         "sum_of_launches_ms": sum_launch},
                "note": "per-launch times from the library's launch log (CUDA events on the launching "
                        "stream, sustained regime); traffic = ncu dram read+write per token-head "
                        "(profiles/ncu_summary.json) scaled to this shape"}

    # ---------------- parity spot check of the timed configuration (two heads)
    parity = None
    if not args.no_parity and rank == 0:
        qg, kg, vg = (t.detach().clone().requires_grad_() for t in (q, k, v))
        o = la2.lightning_attn2(qg, kg, vg, decay)
        o.backward(do)
        torch.cuda.synchronize()
        picks = [(0, 0), (B - 1, H - 1)]
        heads = []
        for b, h in picks:
            f64 = lambda t: t[b, h].detach().double().cpu().numpy()  # noqa: E731
            heads.append((f"b{b}h{h}", lams[h], f64(q), f64(k), f64(v), f64(do), f64(o), f64(qg.grad),
                          f64(kg.grad), f64(vg.grad)))
        del qg, kg, vg, o
        parity = parity_spot_check(heads)

    # ---------------- sweep 1K..64K, each point in the same sustained regime
    sweep = []
    if not args.no_sweep:
        del q, k, v, do
        torch.cuda.empty_cache()
        n = 1024
        while n <= N:
            qs, ks, vs, dos = make(n, n)
            reps = max(5, min(50, (1 << 22) // n))
            t, _ = time_steps(lambda: step(qs, ks, vs, dos), reps, 3, soak_s=args.soak_s)
            fwdf, bwdf = canonical_flops(n, D, D)
            sweep.append({"seq_len": n, "ms": t, "tokens_per_s": B * n * world / (t / 1e3),
                          "tflops": (fwdf + bwdf) * B * H * world / (t / 1e3) / 1e12,
                          "us_per_token": t * 1e3 / n})
            del qs, ks, vs, dos
            n *= 2
        torch.cuda.empty_cache()
        per_tok = [s["us_per_token"] for s in sweep]
        times = [s["ms"] for s in sweep]
        ratios = [b / a for a, b in zip(times, times[1:])]
        flat = {"per_token_max_over_min": max(per_tok) / min(per_tok), "doubling_ratios": ratios}
    else:
        flat = None

    # ---------------- e2e through the public API: pinned host inputs in, o and the
    # gradients back to pinned host buffers, every step. The host link is full duplex, so
    # the steps are software-pipelined like a training loop's data path: step s+1's inputs
    # go up on a copy stream while step s computes, and step s's results come down on a
    # second copy stream (double-buffered device inputs and pinned outputs).
    e2e = None
    if not args.no_e2e:
        host = [t.cpu().pin_memory() for t in make(N, 7)]
        h2d = sum(t.numel() * t.element_size() for t in host)
        # one set of pinned result buffers (the downloads are ordered on one stream); two
        # device input sets so step s+1's upload overlaps step s
        outs = [torch.empty_like(host[0]).pin_memory() for _ in range(4)]
        d2h = sum(t.numel() * t.element_size() for t in outs)
        dev_in = [[torch.empty_like(t, device=dev) for t in host] for _ in range(2)]
        s_up, s_down, s_comp = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.current_stream()
        ev_in = [torch.cuda.Event() for _ in range(2)]     # inputs of set b landed
        ev_used = [torch.cuda.Event() for _ in range(2)]   # compute done reading set b
        ev_out = [torch.cuda.Event() for _ in range(2)]    # results of the step in set b ready

        def upload(b):
            s_up.wait_event(ev_used[b])
            with torch.cuda.stream(s_up):
                for dst, src in zip(dev_in[b], host):
                    dst.copy_(src, non_blocking=True)
                ev_in[b].record(s_up)

        def e2e_run(steps):
            upload(0)
            for st in range(steps):
                b = st & 1
                if st + 1 < steps:
                    upload(1 - b)
                s_comp.wait_event(ev_in[b])
                qh, kh, vh = (t.detach().requires_grad_() for t in dev_in[b][:3])
                o = la2.lightning_attn2(qh, kh, vh, decay)
                o.backward(dev_in[b][3])
                ev_used[b].record(s_comp)
                res = (o.detach(), qh.grad, kh.grad, vh.grad)
                ev_out[b].record(s_comp)
                s_down.wait_event(ev_out[b])
                with torch.cuda.stream(s_down):
                    for dst, src in zip(outs, res):
                        src.record_stream(s_down)
                        dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()

        e2e_run(2)
        barrier()
        torch.cuda.synchronize()
        e2e_steps = max(4, min(args.steps, 16))  # the pipeline fill (first upload) amortised
        t0 = time.perf_counter()
        e2e_run(e2e_steps)
        barrier()
        t_e2e = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
        link = (h2d + d2h) / t_e2e / 1e9
        e2e = {"value": tokens_step / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3, "steps": e2e_steps,
               "host_link_gbs": link,
               "bound": f"host link: {h2d / 2**30:.1f} GiB up + {d2h / 2**30:.1f} GiB down per step "
                        f"({link:.0f} GB/s both directions together) vs {ms:.2f} ms of device time",
               "api": "paper_2401_04658_b200.lightning_attn2 autograd fwd+bwd; q,k,v,dO from pinned "
                      "host, o,dq,dk,dv back to pinned host; uploads / downloads on two copy streams "
                      "overlapping the neighbouring steps (software pipeline, 2 device input sets)"}
        del dev_in, outs, host

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        cb = cpu_reference(N, D, B * H, B * N, args.cpu_sample_heads, reps=3)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {"metric": METRIC if D == 64 else METRIC.replace("d=64", f"d={D}"), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": config, "tflops": tflops,
                "burst": {"ms_per_step": ms_burst, "tokens_per_s": tokens_step / (ms_burst / 1e3),
                          "note": "K steps on a rested GPU (before the power soak)"},
                "sustained_window": soak,
                "roofline": roofline, "parity": parity, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches_per_step * args.steps, "clocks": clk,
                "sweep": sweep, "flatness": flat}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------- other BASELINE configs
def extra_workload(args, world, rank, local_rank):
    """c1: B=1 H=8 N=2048 d=64 (fp32 SIMT path + bf16);  c3: B=32 H=16 N=16K d=128
    (B split over ranks: strong scaling);  c4: B=4 H=20 N=16K d=128 fwd+bwd plus
    recurrent decode (batch 64, 256 graph-captured steps, fp32 state);  c5: one
    512K-token sequence, H=16 d=128 -- intra-GPU sequence split on one GPU,
    sequence parallel (one chunk per rank, state exchange over NCCL) under torchrun."""
    import torch
    import torch.distributed as dist

    import paper_2401_04658_b200 as la2

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    hbm_peak, tc_peak, peak_src = load_peaks()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed_phase(fn, reps=5):
        """Device time of one phase (CUDA events, max over ranks); fn returns nothing."""
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / reps)

    def timed(fn, steps, warmup=3):
        for _ in range(warmup):
            fn()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return max_over_ranks(e0.elapsed_time(e1) / steps)

    def rand(shape, dtype, seed):
        g = torch.Generator(device=dev).manual_seed(seed + 1000 * rank)
        return (torch.rand(*shape, device=dev, generator=g) * 2 - 1).to(dtype)

    w = args.workload
    line = {"n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "higher_is_better": True,
            "vs_baseline": None, "data": "synthetic", "peak_source": peak_src}
    clocks = ClockSampler(local_rank).start()
    if w in ("c1", "c3", "c4"):
        if w == "c1":
            B, H, N, D, dtypes = 1, 8, 2048, 64, (torch.float32, torch.bfloat16)
            decay = [0.5, 0.8, 0.9, 0.95, 0.99, 0.999, 0.9999, 1.0]
        elif w == "c3":
            B, H, N, D, dtypes = max(1, 32 // world), 16, 16384, 128, (torch.bfloat16,)
            decay = alibi_decay(H)
        else:
            B, H, N, D, dtypes = 4, 20, 16384, 128, (torch.bfloat16,)
            decay = alibi_decay(H)
        dec = la2.decay_tensor(decay, H, dev)
        results = {}
        for dt in dtypes:
            q, k, v, do = (rand((B, H, N, D), dt, i) for i in range(4))

            q.requires_grad_(); k.requires_grad_(); v.requires_grad_()

            def step():
                q.grad = k.grad = v.grad = None  # gradients are written, not accumulated
                o = la2.lightning_attn2(q, k, v, dec)
                o.backward(do)
            ms = timed(step, args.steps)
            ff, fb = canonical_flops(N, D, D)
            bf, bb = canonical_bytes(N, D, D, e=2 if dt == torch.bfloat16 else 4)
            results[str(dt).split(".")[-1]] = {
                "ms_per_step": ms, "tokens_per_s": B * N * world / (ms / 1e3),
                "tflops": (ff + fb) * B * H * world / (ms / 1e3) / 1e12,
                "frac_of_roof": max((ff + fb) * B * H / (tc_peak * 1e12), (bf + bb) * B * H / (hbm_peak * 1e9)) * 1e3 / ms}
            q.grad = k.grad = v.grad = None
            del q, k, v, do
        if w == "c1" and rank == 0 and not args.no_cpu:
            # the C1 shape on the host, single core (the reference README
            # methodology) and on all cores, beside the GPU rows
            t_one = statistics.median([_cpu_head_task((N, D, 2000 + r, decay[r % H])) for r in range(3)])
            cb = cpu_reference(N, D, B * H, B * N, B * H)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"]["single_core_tokens_per_s"] = B * N / (t_one * B * H)
        # the config's own dtype: C1 is the reference's fp32 case (BASELINE configs[0]);
        # its bf16 tensor-core time is reported beside it in per_dtype
        main_dt = "float32" if w == "c1" else ("bfloat16" if "bfloat16" in results else "float32")
        line.update({"metric": f"{w} fwd+bwd tokens/s", "value": results[main_dt]["tokens_per_s"],
                     "unit": UNIT, "ms_per_step": results[main_dt]["ms_per_step"],
                     "scaling": "strong" if w == "c3" else "weak", "dtype": "bf16" if main_dt == "bfloat16" else "fp32",
                     "config": {"workload": w, "batch_per_gpu": B, "heads": H, "seq_len": N, "head_dim": D,
                                "api": "lightning_attn2 autograd"},
                     "per_dtype": results})
        if w == "c4":
            # Recurrent decode (tila.inference_step): one launch per token, graph-captured.
            # Batch 64 keeps the fp32 state (84 MB) L2-resident across steps; batch 256
            # (336 MB) streams it from HBM every step, which is the bandwidth-bound case.
            line["decode"] = []
            for Bd in (64, 256):
                steps_d = 256 if Bd == 64 else 64
                st0 = torch.zeros(Bd, H, D, D, device=dev)
                qd, kd, vd = (rand((steps_d, Bd, H, D), torch.bfloat16, 10 + i) for i in range(3))
                st = st0.clone()
                la2.decode_step(qd[0], kd[0], vd[0], dec, st)  # warm the launch path
                graph = torch.cuda.CUDAGraph()
                st.copy_(st0)
                with torch.cuda.graph(graph):
                    for t in range(steps_d):
                        la2.decode_step(qd[t], kd[t], vd[t], dec, st)
                ms_d = timed(graph.replay, max(3, args.steps // 4), 2)
                state_bytes = Bd * H * D * D * 4 * 2  # fp32 state read + write per step
                gbs = state_bytes * steps_d / (ms_d / 1e3) / 1e9
                line["decode"].append({
                    "batch": Bd, "steps_per_graph": steps_d, "ms_per_graph": ms_d,
                    "us_per_step": ms_d * 1e3 / steps_d,
                    "tokens_per_s": Bd * steps_d * world / (ms_d / 1e3), "state_gbs": gbs,
                    "state_mb": Bd * H * D * D * 4 / 2**20,
                    "residency": "L2" if Bd * H * D * D * 4 < 100 * 2**20 else "HBM",
                    "frac_of_hbm": gbs / hbm_peak})
                del st0, st, qd, kd, vd, graph
            # Multi-token decode (la2_decode_tokens: T tokens per launch, state kept in
            # registers across them): batch 256, the HBM-bound case, where the state
            # crossing HBM once per T tokens is the gain
            line["decode_multi"] = []
            Bd = 256
            st = torch.zeros(Bd, H, D, D, device=dev)
            for T in (4, 8, 16):
                qd, kd, vd = (rand((Bd, H, T, D), torch.bfloat16, 20 + i) for i in range(3))
                ms_d = timed(lambda: la2.decode_tokens(qd, kd, vd, dec, st), max(3, args.steps // 4), 2)
                nbytes = Bd * H * D * D * 4 * 2 + 4 * Bd * H * T * D * 2
                line["decode_multi"].append({
                    "batch": Bd, "tokens_per_launch": T, "us_per_launch": ms_d * 1e3,
                    "tokens_per_s": Bd * T * world / (ms_d / 1e3),
                    "gbs": nbytes / (ms_d / 1e3) / 1e9, "frac_of_hbm": nbytes / (ms_d / 1e3) / 1e9 / hbm_peak})
                del qd, kd, vd
            del st
    else:  # c5
        H, D, N_total = 16, 128, 524288
        L = N_total // world
        dec = la2.decay_tensor([min(1.0, x) for x in alibi_decay(H)], H, dev)
        q, k, v, do = (rand((1, H, L, D), torch.bfloat16, i) for i in range(4))
        q.requires_grad_(); k.requires_grad_(); v.requires_grad_()
        if world == 1:
            g = la2.split_factor(1, H, L, D, D, torch.bfloat16)

            def step():
                q.grad = k.grad = v.grad = None
                o = la2.lightning_attn2(q, k, v, dec)
                o.backward(do)
            mode = f"intra-GPU sequence split x{g}"
        else:
            def step():
                q.grad = k.grad = v.grad = None
                o = la2.sp_lightning_attn2(q, k, v, dec, mode=os.environ.get("LA2_SP_MODE", "allgather"))
                o.backward(do)
            mode = f"sequence parallel x{world} ({os.environ.get('LA2_SP_MODE', 'allgather')}) "
        ms = timed(step, args.steps)
        phases = c5_phases(q.detach(), k.detach(), v.detach(), do, dec, world, timed_phase)
        if world == 1:
            # one rank's local work of the 8-GPU run (64K tokens, split into sub-chunks inside
            # the GPU, carried states from the exchange), without the exchange itself
            from paper_2401_04658_b200.sp import cuda_ops
            L8 = N_total // 8
            q8, k8, v8, do8 = (t.detach()[:, :, :L8].contiguous() for t in (q, k, v, do))
            local = cuda_ops("auto")
            kv8 = local.chunk_state(k8, v8, dec)
            dkv8 = local.chunk_dstate(q8, do8, dec)

            def rank_step():
                local.chunk_state(k8, v8, dec)
                local.forward(q8, k8, v8, dec, kv8)
                local.chunk_dstate(q8, do8, dec)
                local.backward(q8, k8, v8, do8, dec, kv8, dkv8)
            ms8 = timed(rank_step, args.steps)
            phases["sp8_rank_local"] = {"tokens": L8, "sub_chunks": local.split.get("g", 1),
                                        "ms_fwd_bwd": ms8, "fraction_of_1gpu_step": ms8 / ms,
                                        "note": "one rank's local passes A+B fwd+bwd of the 8-GPU "
                                                "sequence-parallel run (exchange excluded)"}
            del q8, k8, v8, do8
        ff, fb = canonical_flops(N_total, D, D)
        bf, bb = canonical_bytes(N_total, D, D)
        line.update({"metric": "c5 fwd+bwd tokens/s (one 512K sequence)", "value": N_total / (ms / 1e3),
                     "unit": UNIT, "ms_per_step": ms, "scaling": "strong", "dtype": "bf16",
                     "config": {"workload": "c5", "seq_len": N_total, "heads": H, "head_dim": D,
                                "per_rank_tokens": L, "mode": mode},
                     "phases_ms": phases,
                     "tflops": (ff + fb) * H / (ms / 1e3) / 1e12,
                     "frac_of_roof": max((ff + fb) * H / (tc_peak * 1e12 * world),
                                         (bf + bb) * H / (hbm_peak * 1e9 * world)) * 1e3 / ms})
    line["clocks"] = clocks.stop()
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
