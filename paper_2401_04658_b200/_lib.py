"""ctypes binding of the C ABI in ``include/la2.h`` (``libla2.so``, built in-tree).

There is no fallback: if the library is missing or cannot be loaded, importing
the ops raises. Errors returned by the ABI map to ValueError (argument /
unsupported shape, like the reference's ValueError cases in
pkg/src/tila/reference.py:42-74) or RuntimeError (CUDA failures).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("LA2_LIB", _PKG / "libla2.so"))

LA2_BF16 = 0
LA2_FP32 = 1
LA2_ERR_VALUE = -1
LA2_ERR_UNSUPPORTED = -2
LA2_ERR_CUDA = -3

_vp = ctypes.c_void_p
_i = ctypes.c_int


class LaunchRecord(ctypes.Structure):
    """struct la2_launch_record (include/la2.h)."""
    _fields_ = [("kernel", ctypes.c_char * 48), ("grid", ctypes.c_int), ("cluster", ctypes.c_int),
                ("ms", ctypes.c_float)]


# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "la2_version": [],
    "la2_last_error": [],
    "la2_forward": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_forward_strided": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i,
                            ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, _vp],
    "la2_backward": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_backward_strided": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i,
                             ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, _vp],
    "la2_chunk_state": [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_chunk_dstate": [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_state_scan": [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, ctypes.POINTER(ctypes.c_int), _i, _vp],
    "la2_decode_step": [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp],
    "la2_decode_tokens": [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_check_decay": [_vp, _i, _vp],
    "la2_state_blocks_bytes": [_i, _i, _i, _i, _i],
    "la2_forward_states": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_backward_states": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i,
                            _vp],
    "la2_forward_f64": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_backward_f64": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_decode_step_f64": [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp],
    "la2_decode_tokens_f64": [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp],
    "la2_check_decay_f64": [_vp, _i, _vp],
    "la2_forward_norm": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_float, _i, _i, _i, _i, _i, _i,
                         _i, _vp],
    "la2_rmsnorm_forward": [_vp, _vp, _vp, _i, _i, _i, _i, _i, ctypes.c_float, _i, _vp],
    "la2_rmsnorm_backward": [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp],
    "la2_launch_log": [_i],
    "la2_launch_log_read": [ctypes.POINTER(LaunchRecord), _i],
    "la2_set_tuning": [_i, _i],
    "la2_workspace_bytes": [],
}
_RESTYPES = {"la2_last_error": ctypes.c_char_p, "la2_workspace_bytes": ctypes.c_longlong,
             "la2_state_blocks_bytes": ctypes.c_longlong,
             "la2_dev_last_error": ctypes.c_char_p}
_DEV_ONLY = {"la2_set_tuning"}

# development library (include/la2_dev.h): not the shipping ABI
DEV_LIB_PATH = _PKG / "libla2_dev.so"
DEV_SIGNATURES: dict[str, list] = {
    "la2_dev_last_error": [],
    "la2_selftest_umma": [_vp, _vp, _vp, _i, _i, _i, _i, _i, _vp],
    "la2_bench_umma": [_i, _i, _i, _i, _i, _i, _vp, _vp],
    "la2_bench_tmem": [_i, _i, _i, _i, _vp, _vp, _vp],
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libla2.so once; raise ImportError (loudly) if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -m paper_2401_04658_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, args in SIGNATURES.items():
        if name in _DEV_ONLY and not hasattr(lib, name):
            continue  # development entry points (older or trimmed builds)
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = load().la2_last_error().decode(errors="replace")
    if rc in (LA2_ERR_VALUE, LA2_ERR_UNSUPPORTED):
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (code {rc})")


_fns: dict = {}


def call(name: str, *args) -> None:
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(load(), name)
    rc = fn(*args)
    if rc:
        check(rc, name)


_dev = None


def load_dev() -> ctypes.CDLL:
    """Load the development library libla2_dev.so (self-test and micro-benchmarks)."""
    global _dev
    if _dev is not None:
        return _dev
    if not DEV_LIB_PATH.exists():
        raise ImportError(f"{DEV_LIB_PATH} not found: build it with `python -m paper_2401_04658_b200.build`")
    lib = ctypes.CDLL(str(DEV_LIB_PATH))
    for name, args in DEV_SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _dev = lib
    return lib


def call_dev(name: str, *args) -> None:
    lib = load_dev()
    rc = getattr(lib, name)(*args)
    if rc:
        msg = lib.la2_dev_last_error().decode(errors="replace")
        if rc in (LA2_ERR_VALUE, LA2_ERR_UNSUPPORTED):
            raise ValueError(f"{name}: {msg}")
        raise RuntimeError(f"{name}: {msg} (code {rc})")
