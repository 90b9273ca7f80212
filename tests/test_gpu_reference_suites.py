"""The reference's own gating suites, run against the GPU kernels.

The unmodified reference package ``tila`` is installed (test infrastructure only, git-
ignored) into ``baseline/_ref`` by

    python -m pip install --no-index --no-build-isolation --no-deps \\
        --target baseline/_ref <copy of /root/reference/pkg>

``tila.verify`` imports its kernels by name (pkg/src/tila/verify.py:17), so patching
``tila.verify.tiled_forward / tiled_backward / chunked_forward`` with the GPU-backed
``paper_2401_04658_b200.tila_api`` functions (same signatures) makes
``run_equivalence_suite`` and ``run_gradcheck_suite`` (verify.py:212-263) exercise the
CUDA path on their normative grids, against the reference's own oracles (masked product,
per-token recurrence, central finite differences) computed by the reference itself.
The GPU computes in fp32, so the gate is the north star's fp32 tolerance 1e-4 instead
of the suites' fp64 1e-10 / 1e-5.
"""

import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
FP32_TOL = 1e-4


@pytest.fixture(scope="module")
def tila_gpu():
    if not (REF / "tila" / "verify.py").exists():
        pytest.skip("reference package not installed in baseline/_ref (see module docstring)")
    sys.path.insert(0, str(REF))
    try:
        import tila
        import tila.verify as verify
    finally:
        sys.path.remove(str(REF))
    assert Path(tila.__file__).resolve().is_relative_to(REF.resolve()), tila.__file__
    from paper_2401_04658_b200 import tila_api

    saved = {n: getattr(verify, n) for n in ("tiled_forward", "tiled_backward", "chunked_forward")}
    verify.tiled_forward = tila_api.tiled_forward
    verify.tiled_backward = tila_api.tiled_backward
    verify.chunked_forward = tila_api.chunked_forward
    try:
        yield verify
    finally:
        for n, f in saved.items():
            setattr(verify, n, f)


def _summary(reports):
    worst = max(reports, key=lambda r: r.max_rel_error)
    fails = [str(r) for r in reports if not r.passed]
    return worst, fails


def test_reference_equivalence_suite_small_grid(tila_gpu):
    v = tila_gpu
    cfg = v.SuiteConfig(cases=v.small_grid().cases, tolerance=FP32_TOL)
    reports = v.run_equivalence_suite(cfg)
    worst, fails = _summary(reports)
    print(f"{len(reports)} comparisons, worst: {worst}")
    assert len(reports) == 7 * len(cfg.cases)
    assert not fails, fails[:10]


def test_reference_equivalence_suite_default_grid(tila_gpu):
    """The normative grid (verify.py:127-138: n up to 256, d in {1, 4, 32}, dv = d or
    d + 3, blocks 1..64, lam in {0.5, 0.9, 0.999, 1}), every case."""
    v = tila_gpu
    cfg = v.SuiteConfig(cases=v.default_grid().cases, tolerance=FP32_TOL)
    reports = v.run_equivalence_suite(cfg)
    worst, fails = _summary(reports)
    print(f"{len(reports)} comparisons, worst: {worst}")
    assert len(cfg.cases) == 1536
    assert not fails, fails[:10]


def test_reference_gradcheck_suite(tila_gpu):
    """GPU tiled backward against the reference's central finite differences."""
    v = tila_gpu
    cfg = v.SuiteConfig(cases=v.default_gradcheck_grid().cases, tolerance=FP32_TOL)
    reports = v.run_gradcheck_suite(cfg)
    worst, fails = _summary(reports)
    print(f"{len(reports)} comparisons, worst: {worst}")
    assert not fails, fails[:10]
