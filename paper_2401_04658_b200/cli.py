"""Operator CLI for the B200 path, mirroring the reference's ``tila`` CLI
(pkg/src/tila/cli.py:45-202): ``verify``, ``gradcheck``, ``bench``, ``sweep-block``,
``stream-demo`` with the same flags and exit codes (0 pass, 1 fail, 2 usage).

The checks run on the GPU against an fp64 *quadratic* restatement of the op computed
with torch on the same device -- ``O = ((Q Kᵀ) ⊙ M) V`` with ``M[t,s] = λ^(t-s)``, the
reference's ``oracle_forward`` / ``oracle_backward`` formulation
(pkg/src/tila/reference.py:118-132, :184-204) -- so the tool needs no CPU reference and
runs on the GPU box as is. The error metric is the reference's
``max|cand - ref| / max|ref|`` (pkg/src/tila/verify.py:50-75).

    python -m paper_2401_04658_b200.cli verify --grid small
    python -m paper_2401_04658_b200.cli bench --impls tiled,chunked --lens 1024,2048,4096,8192 --dim 64 --block 64
"""

from __future__ import annotations

import argparse
import sys
from dataclasses import dataclass

import torch

from . import gpubench, ops

BENCH_LAMBDA = 0.9
TOL = {torch.float32: 1e-4, torch.bfloat16: 1e-2}


def _int_list(text: str) -> list:
    try:
        return [int(tok) for tok in text.split(",") if tok]
    except ValueError as e:
        raise argparse.ArgumentTypeError(str(e)) from None


def _str_list(text: str) -> list:
    return [tok for tok in text.split(",") if tok]


@dataclass
class Report:
    label: str
    max_rel_error: float
    tolerance: float

    @property
    def passed(self) -> bool:
        return self.max_rel_error <= self.tolerance

    def __str__(self) -> str:
        return f"{self.label}: max rel {self.max_rel_error:.3e} (tol {self.tolerance:g})"


def rel_err(cand: torch.Tensor, ref: torch.Tensor) -> float:
    ref = ref.double()
    return float((cand.double() - ref).abs().max() / max(float(ref.abs().max()), 1e-12))


def quadratic_reference(q, k, v, lam: torch.Tensor):
    """fp64 masked quadratic attention per (b, h): the reference oracle's formulation."""
    n = q.shape[2]
    t = torch.arange(n, device=q.device, dtype=torch.float64)
    diff = t[:, None] - t[None, :]
    lg = torch.log(lam.double()).view(1, -1, 1, 1)
    mask = torch.where(diff >= 0, torch.exp(lg * diff.clamp(min=0)), torch.zeros((), dtype=torch.float64,
                                                                                device=q.device))
    s = torch.einsum("bhtd,bhsd->bhts", q.double(), k.double()) * mask
    return torch.einsum("bhts,bhsv->bhtv", s, v.double())


def _inputs(B, H, n, d, dv, dtype, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    mk = lambda c: (torch.rand(B, H, n, c, device=dev, generator=g, dtype=torch.float64) * 2 - 1).to(dtype)
    return mk(d), mk(d), mk(dv), mk(dv)


def _grid(name: str):
    ns = (1, 2, 7, 16, 33, 64, 100, 256) if name == "small" else (1, 2, 7, 16, 33, 64, 100, 256, 1000, 4096)
    lams = (0.5, 0.9, 0.999, 1.0)
    shapes = [(torch.float32, 4, 7), (torch.float32, 32, 35), (torch.bfloat16, 64, 64),
              (torch.bfloat16, 128, 128)]
    if name == "default":
        shapes += [(torch.float32, 64, 64), (torch.bfloat16, 64, 128), (torch.bfloat16, 128, 64)]
    return ns, lams, shapes


def run_equivalence(grid: str, seeds, tol_override=None) -> list:
    dev = torch.device("cuda", torch.cuda.current_device())
    ns, lams, shapes = _grid(grid)
    reports = []
    for dtype, d, dv in shapes:
        tol = tol_override if tol_override is not None else TOL[dtype]
        for n in ns:
            for seed in seeds:
                q, k, v, do = _inputs(1, len(lams), n, d, dv, dtype, seed, dev)
                lam = torch.tensor(lams, dtype=torch.float32, device=dev)
                ref = quadratic_reference(q, k, v, lam)
                tag = f"{str(dtype).split('.')[-1]} d={d} dv={dv} n={n} seed={seed}"
                o, kv = ops.la2_forward(q, k, v, lam, output_final_state=True)
                reports.append(Report(f"tiled {tag}", rel_err(o, ref), tol))
                # chunked: three ragged chunks with the carried state (kernel.py:142-162)
                cuts = sorted({0, n // 3, (2 * n) // 3 + (1 if n > 2 else 0), n})
                state, outs = None, []
                for a, b in zip(cuts, cuts[1:]):
                    if b > a:
                        oc, state = ops.la2_forward(q[:, :, a:b], k[:, :, a:b], v[:, :, a:b], lam,
                                                    kv_in=state, output_final_state=True)
                        outs.append(oc)
                reports.append(Report(f"chunked {tag}", rel_err(torch.cat(outs, 2), ref), tol))
                reports.append(Report(f"chunked final state {tag}", rel_err(state, kv), tol))
                # the per-token recurrence, all n tokens in one launch (reference.py:142-159)
                rec, rst = ops.recurrent_forward(q, k, v, lam)
                reports.append(Report(f"recurrent {tag}", rel_err(rec, ref), tol))
                reports.append(Report(f"recurrent final state {tag}", rel_err(rst, kv), tol))
                grads = ops.la2_backward(q, k, v, do, lam)[:3]
                for name, g, rg in zip(("dq", "dk", "dv"), grads, _ref_grads(q, k, v, do, lam)):
                    reports.append(Report(f"backward {name} {tag}", rel_err(g, rg), tol))
    return reports


def _ref_grads(q, k, v, do, lam):
    qd, kd, vd = (t.detach().double().requires_grad_() for t in (q, k, v))
    out = quadratic_reference(qd, kd, vd, lam)
    return torch.autograd.grad(out, (qd, kd, vd), do.double())


def _print_reports(reports, kind: str) -> int:
    failed = [r for r in reports if not r.passed]
    worst = max(reports, key=lambda r: r.max_rel_error / r.tolerance) if reports else None
    print(f"{kind}: {len(reports)} comparisons, {len(failed)} failed")
    if worst is not None:
        print(f"worst {worst}")
    for r in failed[:10]:
        print(f"  {r}")
    if len(failed) > 10:
        print(f"  ... and {len(failed) - 10} more failures")
    return 0 if not failed else 1


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="la2", description="B200 Lightning-2: verification and benchmarks.")
    sub = parser.add_subparsers(dest="command", required=True)
    p_verify = sub.add_parser("verify", help="forward/backward equivalence suite on the GPU")
    p_verify.add_argument("--tolerance", type=float, default=None,
                          help="override the per-dtype gate (1e-4 fp32, 1e-2 bf16)")
    p_verify.add_argument("--seed", type=int, default=None)
    p_verify.add_argument("--grid", choices=("default", "small"), default="small")
    p_grad = sub.add_parser("gradcheck", help="GPU gradients against fp64 autograd of the quadratic form")
    p_grad.add_argument("--epsilon", type=float, default=1e-6, help="accepted for CLI parity; unused")
    p_bench = sub.add_parser("bench", help="sequence-length scaling sweep, writes CSV")
    p_bench.add_argument("--impls", type=_str_list, required=True)
    p_bench.add_argument("--lens", type=_int_list, required=True)
    p_bench.add_argument("--dim", type=int, required=True)
    p_bench.add_argument("--block", type=int, required=True)
    p_bench.add_argument("--reps", type=int, default=5)
    p_bench.add_argument("--heads", type=int, default=1)
    p_bench.add_argument("--out", default="bench.csv")
    p_sweep = sub.add_parser("sweep-block", help="block-size sweep at fixed length")
    p_sweep.add_argument("--len", dest="length", type=int, required=True)
    p_sweep.add_argument("--dim", type=int, required=True)
    p_sweep.add_argument("--blocks", type=_int_list, required=True)
    p_sweep.add_argument("--reps", type=int, default=5)
    p_sweep.add_argument("--out", default=None)
    p_stream = sub.add_parser("stream-demo", help="streaming inference over carried state")
    p_stream.add_argument("--dim", type=int, required=True)
    p_stream.add_argument("--chunk", type=int, required=True)
    p_stream.add_argument("--chunks", type=int, required=True)
    p_stream.add_argument("--lambda", dest="lam", type=float, default=BENCH_LAMBDA)
    return parser


def _cmd_verify(args) -> int:
    seeds = [args.seed] if args.seed is not None else [0, 1]
    reports = run_equivalence(args.grid, seeds, args.tolerance)
    return _print_reports(reports, f"equivalence suite ({args.grid} grid, GPU)")


def _cmd_gradcheck(args) -> int:
    reports = []
    dev = torch.device("cuda", torch.cuda.current_device())
    for dtype, d in ((torch.float32, 4), (torch.float32, 64), (torch.bfloat16, 64), (torch.bfloat16, 128)):
        for n in (1, 5, 64, 300):
            q, k, v, do = _inputs(1, 2, n, d, d, dtype, 7, dev)
            lam = torch.tensor([0.9, 1.0], device=dev)
            for name, g, rg in zip(("dq", "dk", "dv"), ops.la2_backward(q, k, v, do, lam)[:3],
                                   _ref_grads(q, k, v, do, lam)):
                reports.append(Report(f"{name} {str(dtype).split('.')[-1]} d={d} n={n}", rel_err(g, rg), TOL[dtype]))
    return _print_reports(reports, "gradcheck suite (GPU vs fp64 autograd)")


def _cmd_bench(args, parser) -> int:
    for impl in args.impls:
        if impl not in gpubench.IMPLS:
            parser.error(f"unknown impl {impl!r}, expected one of {','.join(gpubench.IMPLS)}")
    if len(args.lens) < 4:
        parser.error("minimum 4 points required in --lens")
    for a, b in zip(args.lens, args.lens[1:]):
        if b != 2 * a:
            parser.error(f"--lens must strictly double, got {a} -> {b}")
    records, verdicts = gpubench.scaling_sweep(args.impls, args.lens, d=args.dim, block=args.block,
                                               lam=BENCH_LAMBDA, reps=args.reps, heads=args.heads)
    gpubench.emit_csv(records, args.out)
    print(f"wrote {len(records)} records to {args.out}")
    for r in records:
        print(f"  {r.impl:10s} {r.direction:8s} n={r.n:<7d} median={r.median_seconds:.6f}s "
              f"us/token={r.per_token_microseconds:.3f} scratch={r.scratch_bytes}")
    code = 0
    for v in verdicts:
        print(f"{v.impl}: ratios [{', '.join(f'{x:.2f}' for x in v.ratios)}] -> {v.classification}")
        if v.impl == "tiled" and v.classification != "linear-like":
            code = 1
    return code


def _cmd_sweep_block(args) -> int:
    records = gpubench.block_size_sweep(args.length, args.dim, BENCH_LAMBDA, args.blocks, args.reps)
    if args.out:
        gpubench.emit_csv(records, args.out)
        print(f"wrote {len(records)} records to {args.out}")
    for r in records:
        print(f"  B={r.block:<6d} median={r.median_seconds:.6f}s us/token={r.per_token_microseconds:.3f} "
              f"scratch={r.scratch_bytes}")
    fastest = min(records, key=lambda r: r.median_seconds)
    print(f"fastest block size on this GPU: {fastest.block} (the kernel's own tile is 128 tokens)")
    return 0


def _cmd_stream_demo(args) -> int:
    d, chunk, chunks, lam = args.dim, args.chunk, args.chunks, args.lam
    dev = torch.device("cuda", torch.cuda.current_device())
    dtype = torch.bfloat16 if d in (64, 128) else torch.float32
    total = chunk * chunks
    q, k, v, _ = _inputs(1, 1, total, d, d, dtype, 0, dev)
    lam_t = torch.tensor([lam], device=dev)
    state, outs = None, []
    for i in range(chunks):
        sl = slice(i * chunk, (i + 1) * chunk)
        o, state = ops.la2_forward(q[:, :, sl], k[:, :, sl], v[:, :, sl], lam_t, kv_in=state,
                                   output_final_state=True)
        outs.append(o)
    streamed = torch.cat(outs, 2)
    print(f"streamed {chunks} chunks of {chunk} tokens (d={d}, lambda={lam}, {str(dtype).split('.')[-1]}); "
          f"tokens absorbed: {total}")
    print(f"final state checksum: {float(state.double().sum()):.12e}")
    # one-shot recompute by the per-token recurrence, as the reference's demo does
    # (pkg/src/tila/cli.py:179: recurrent_forward)
    one_shot, ref_state = ops.recurrent_forward(q, k, v, lam_t)
    tol = TOL[dtype]
    e_o, e_s = rel_err(streamed, one_shot), rel_err(state, ref_state)
    ok = e_o <= tol and e_s <= tol
    print(f"one-shot recompute max rel error: outputs {e_o:.3e}, state {e_s:.3e} -> "
          f"{'match' if ok else 'MISMATCH'}")
    return 0 if ok else 1


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    if args.command == "verify":
        return _cmd_verify(args)
    if args.command == "gradcheck":
        return _cmd_gradcheck(args)
    if args.command == "bench":
        return _cmd_bench(args, parser)
    if args.command == "sweep-block":
        return _cmd_sweep_block(args)
    if args.command == "stream-demo":
        return _cmd_stream_demo(args)
    parser.error(f"unknown command {args.command!r}")
    return 2


if __name__ == "__main__":
    sys.exit(main())
