"""Recipe: stage the reference package itself under ``oracle/_ref/`` (TEST INFRASTRUCTURE).

The reference (``/root/reference/pkg/src/tila``) is pure Python/NumPy, so "building"
it is copying the unmodified package into ``oracle/_ref/tila`` -- a git-ignored
directory that travels to the GPU box with the repo snapshot (``/root/reference``
does not exist there). ``tests/test_gpu_reference_suites.py`` imports it from there
to run the reference's own gating suites (``verify.run_equivalence_suite``,
``verify.run_gradcheck_suite``, pkg/src/tila/verify.py:212-263) with the GPU kernels
patched in as the candidate implementation, exactly as INTEGRATION.md describes.

Nothing in the product package reads ``oracle/_ref``. No reference source is committed.
"""

from __future__ import annotations

import shutil
from pathlib import Path

REF_PKG = Path("/root/reference/pkg/src/tila")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent / "_ref"


def build(out: Path = OUT) -> Path | None:
    """Copy the reference package to ``out/tila`` when the reference is present (this
    container); return the staged path, or None (e.g. on the GPU box, which only uses
    what a previous build staged)."""
    if not (REF_PKG / "verify.py").exists():
        return (out / "tila") if (out / "tila" / "verify.py").exists() else None
    dst = out / "tila"
    out.mkdir(parents=True, exist_ok=True)
    shutil.copytree(REF_PKG, dst, dirs_exist_ok=True,
                    ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    # the reference's own test suite, run against the GPU adapter by
    # tests/test_gpu_reference_suites.py (tests/ref_gpu_plugin.py patches the kernels in)
    if REF_TESTS.is_dir():
        shutil.copytree(REF_TESTS, out / "tests", dirs_exist_ok=True,
                        ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    return dst


if __name__ == "__main__":
    print(build())
