"""Build the C-ABI library ``libla2.so`` in-tree for sm_100a.

Plain ``nvcc -shared`` (static cudart), no torch headers: the library exposes
only the C ABI declared in ``include/la2.h``. Run ``python -m
paper_2401_04658_b200.build`` or call :func:`build`.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libla2.so"
SOURCES = ["la2_api.cu", "la2_tc.cu", "la2_simt.cu", "la2_f64.cu", "la2_norm.cu"]
# development library (include/la2_dev.h): operand-layout self-test and micro-benchmarks
DEV_LIB = PKG / "libla2_dev.so"
DEV_SOURCES = ["la2_selftest.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _flags() -> list[str]:
    return ARCH + [
        "-O3", "-lineinfo", "-std=c++17", "--use_fast_math", "-Xcompiler", "-fPIC",
        "-Xcompiler", "-fvisibility=hidden", f"-I{ROOT / 'include'}", f"-I{CSRC}",
    ]


def _compile(src: str, verbose: bool, extra=(), tag="") -> Path:
    obj = CSRC / (Path(src).stem + tag + ".o")
    cmd = [NVCC, *_flags(), *extra, "-c", str(CSRC / src), "-o", str(obj)]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr, file=sys.stderr)
    return obj


def _stale(lib: Path, sources) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in sources] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps += list((ROOT / "include").glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> Path:
    """Build libla2.so and libla2_dev.so (or, with trace=True, the phase-trace variant
    libla2_trace.so). Returns the path of libla2.so."""
    if not trace:
        _link(DEV_LIB, DEV_SOURCES, force, verbose, (), "")
        return _link(LIB, SOURCES, force, verbose, (), "")
    return _link(PKG / "libla2_trace.so", SOURCES, True, verbose, ["-DLA2_TRACE"], "_trace")


def _link(lib: Path, sources, force: bool, verbose: bool, extra, tag) -> Path:
    if not force and not _stale(lib, sources):
        return lib
    extra = [*extra, *os.environ.get("LA2_NVCC_EXTRA", "").split()]
    with cf.ThreadPoolExecutor(len(sources)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, extra, tag), sources))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, lib)
    for o in objs:
        o.unlink(missing_ok=True)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
