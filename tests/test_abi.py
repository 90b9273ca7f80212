"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/la2.h declares; argument validation returns the documented error
codes before any device work. CPU only (no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "la2.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"LA2_API\s+[\w\s\*]+?\b(la2_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2401_04658_b200 import build, _lib

    build.build()
    return _lib.load()


def test_header_declares_entry_points():
    syms = declared_symbols()
    for name in ("la2_forward", "la2_backward", "la2_chunk_state", "la2_chunk_dstate",
                 "la2_state_scan", "la2_decode_step", "la2_last_error", "la2_version"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_python_binding_covers_header(lib):
    from paper_2401_04658_b200 import _lib

    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_version(lib):
    assert lib.la2_version() == 100


def test_validation_errors_without_device(lib):
    from paper_2401_04658_b200 import _lib

    dummy = ctypes.c_void_p(16)
    # N = 0 -> LA2_ERR_VALUE (the reference rejects empty sequences: matrix.py:56-57)
    rc = lib.la2_forward(dummy, dummy, dummy, dummy, dummy, None, None, 1, 1, 0, 64, 64, 0, None)
    assert rc == _lib.LA2_ERR_VALUE
    assert b"N must be" in lib.la2_last_error()
    # null decay
    rc = lib.la2_forward(dummy, dummy, dummy, None, dummy, None, None, 1, 1, 8, 64, 64, 0, None)
    assert rc == _lib.LA2_ERR_VALUE
    # unsupported dtype
    rc = lib.la2_forward(dummy, dummy, dummy, dummy, dummy, None, None, 1, 1, 8, 64, 64, 7, None)
    assert rc == _lib.LA2_ERR_UNSUPPORTED
    # fp32 with d > 256 is outside both kernels' envelope (no fallback)
    rc = lib.la2_forward(dummy, dummy, dummy, dummy, dummy, None, None, 1, 1, 8, 320, 64, 1, None)
    assert rc == _lib.LA2_ERR_UNSUPPORTED
    assert b"unsupported shape" in lib.la2_last_error()
    rc = lib.la2_backward(dummy, dummy, dummy, dummy, dummy, dummy, dummy, None, None, None, None,
                          1, 1, 8, 64, 64, 0, None)
    assert rc == _lib.LA2_ERR_VALUE
    lens = (ctypes.c_int * 1)(0)
    rc = lib.la2_state_scan(dummy, dummy, None, dummy, 1, 1, 1, 4, 4, lens, 0, None)
    assert rc != 0


def test_check_maps_codes_to_python_errors(lib):
    from paper_2401_04658_b200 import _lib

    with pytest.raises(ValueError):
        _lib.call("la2_forward", 16, 16, 16, 16, 16, None, None, 1, 1, 0, 64, 64, 0, None)


def test_header_is_plain_c_and_links(lib, tmp_path):
    """The boundary is usable from C (what a cgo / JNI / N-API shim compiles against):
    la2.h compiles as C99 with -Wall -Werror and a C program links against libla2.so and
    calls an entry point."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "use_la2.c"
    src.write_text('#include "la2.h"\n#include <stdio.h>\n'
                   'int main(void) { int v = la2_version(); '
                   'int rc = la2_forward(0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 64, 64, LA2_BF16, 0); '
                   'printf("%d %d\\n", v, rc); return (v > 0 && rc == LA2_ERR_VALUE) ? 0 : 1; }\n')
    libdir = ROOT / "paper_2401_04658_b200"
    exe = tmp_path / "use_la2"
    subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", f"-I{ROOT / 'include'}", str(src),
                    f"-L{libdir}", "-l:libla2.so", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout + res.stderr


def test_check_decay_host_memory(lib):
    """la2_check_decay on host memory needs no device: lam in (0, 1] passes, anything
    else is LA2_ERR_VALUE naming the head (reference.py:42-44)."""
    from paper_2401_04658_b200 import _lib

    good = (ctypes.c_float * 3)(0.5, 1.0, 1e-30)
    assert lib.la2_check_decay(good, 3, None) == 0
    for vals in ((0.5, 1.5), (0.5, 0.0), (0.5, -1.0), (0.5, float("nan"))):
        arr = (ctypes.c_float * 2)(*vals)
        assert lib.la2_check_decay(arr, 2, None) == _lib.LA2_ERR_VALUE
        assert b"head 1" in lib.la2_last_error()
    assert lib.la2_check_decay(None, 2, None) == _lib.LA2_ERR_VALUE


def test_dev_library_is_separate(lib):
    """The self-test / micro-benchmark entry points live in libla2_dev.so
    (include/la2_dev.h), not in the shipping libla2.so."""
    from paper_2401_04658_b200 import _lib

    dev = _lib.load_dev()
    text = (ROOT / "include" / "la2_dev.h").read_text()
    dev_syms = set(re.findall(r"LA2_API\s+[\w\s\*]+?\b(la2_\w+)\s*\(", text))
    assert dev_syms == set(_lib.DEV_SIGNATURES)
    for name in dev_syms:
        assert hasattr(dev, name), name
        assert not hasattr(lib, name), name


def test_f64_entry_points_validate_without_device(lib):
    """The double-precision entry points (la2_*_f64) reject bad shapes / nulls before any
    device work, and la2_check_decay_f64 validates host decay like the reference."""
    from paper_2401_04658_b200 import _lib

    dummy = ctypes.c_void_p(16)
    assert lib.la2_forward_f64(dummy, dummy, dummy, dummy, dummy, None, None, 1, 1, 0, 4, 4, 0,
                               None) == _lib.LA2_ERR_VALUE
    assert lib.la2_forward_f64(dummy, dummy, dummy, None, dummy, None, None, 1, 1, 8, 4, 4, 0,
                               None) == _lib.LA2_ERR_VALUE
    assert lib.la2_forward_f64(dummy, dummy, dummy, dummy, dummy, None, None, 1, 1, 8, 300, 4, 0,
                               None) == _lib.LA2_ERR_UNSUPPORTED
    assert lib.la2_backward_f64(dummy, dummy, dummy, dummy, dummy, None, dummy, dummy, None, None, None,
                                1, 1, 8, 4, 4, 0, None) == _lib.LA2_ERR_VALUE
    assert lib.la2_decode_step_f64(dummy, dummy, dummy, dummy, None, dummy, 1, 1, 4, 4,
                                   None) == _lib.LA2_ERR_VALUE
    # multi-token decode: T < 0 rejected, T = 0 a no-op before any device work
    assert lib.la2_decode_tokens_f64(dummy, dummy, dummy, dummy, dummy, dummy, 1, 1, -1, 4, 4,
                                     None) == _lib.LA2_ERR_VALUE
    assert lib.la2_decode_tokens_f64(dummy, dummy, dummy, dummy, dummy, dummy, 1, 1, 0, 4, 4, None) == 0
    assert lib.la2_decode_tokens(dummy, dummy, dummy, dummy, dummy, dummy, 1, 1, -1, 4, 4, _lib.LA2_FP32,
                                 None) == _lib.LA2_ERR_VALUE
    assert lib.la2_decode_tokens(dummy, dummy, dummy, dummy, dummy, dummy, 1, 1, 0, 4, 4, _lib.LA2_FP32,
                                 None) == 0
    assert lib.la2_decode_tokens(dummy, dummy, dummy, dummy, None, dummy, 1, 1, 3, 4, 4, _lib.LA2_FP32,
                                 None) == _lib.LA2_ERR_VALUE
    assert lib.la2_decode_tokens(dummy, dummy, dummy, dummy, dummy, dummy, 1, 1, 3, 4, 4, 7,
                                 None) == _lib.LA2_ERR_UNSUPPORTED
    good = (ctypes.c_double * 3)(0.5, 1.0, 1e-300)
    assert lib.la2_check_decay_f64(good, 3, None) == 0
    for vals in ((0.5, 1.0000000001), (0.5, 0.0), (0.5, float("nan"))):
        arr = (ctypes.c_double * 2)(*vals)
        assert lib.la2_check_decay_f64(arr, 2, None) == _lib.LA2_ERR_VALUE
        assert b"head 1" in lib.la2_last_error()


def test_tensor_core_envelope_documented():
    """The header's kernel-selection rule names the widened bf16 envelope (multiples of 8
    up to 256) and the fp64 entry points."""
    text = HEADER.read_text()
    assert "multiples of 8 up to 256" in text
    assert "la2_forward_f64" in text and "la2_backward_f64" in text


def test_integration_table_covers_header():
    """INTEGRATION.md names every entry point include/la2.h declares (with the reference
    function it replaces, or why it has none)."""
    text = (HEADER.parents[1] / "INTEGRATION.md").read_text()
    missing = [s for s in declared_symbols() if f"`{s}`" not in text and f"{s}`" not in text]
    assert not missing, missing
