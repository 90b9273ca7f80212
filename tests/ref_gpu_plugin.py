"""pytest plugin: run the reference's own test suite (oracle/_ref/tests, staged by
oracle/build_ref.py) with the reference's operator API served by the GPU.

Loaded with ``-p ref_gpu_plugin`` before the reference's test modules import ``tila``:
it replaces tila's public kernel entry points -- tiled_forward, tiled_backward,
chunked_forward, batched_forward, batched_backward, inference_step
(pkg/src/tila/__init__.py:13-40) -- with the GPU adapter
(paper_2401_04658_b200.tila_api), in the ``tila`` namespace the tests import from and in
``tila.verify`` (which imports them by name). Everything else (oracles, recurrence, power
tables, fixtures, CLI, bench) stays the reference's own code, so every kernel-level
assertion of the suite compares the GPU against the reference. With
LA2_REF_PATCH_RECURRENT=1 the per-token recurrence (tila.recurrent_forward) is served by
the GPU too (la2_decode_tokens), so the reference's recurrence tests (test_reference.py)
check the GPU recurrence against its oracle, hand values and the inference_step fold.
TEST INFRASTRUCTURE ONLY.
"""

import os

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT / "oracle" / "_ref", ROOT):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

PATCHED = ("tiled_forward", "tiled_backward", "chunked_forward", "batched_forward", "batched_backward",
           "inference_step")
if os.environ.get("LA2_REF_PATCH_RECURRENT") == "1":
    PATCHED = PATCHED + ("recurrent_forward",)


def pytest_configure(config):
    import tila
    import tila.bench
    import tila.verify

    from paper_2401_04658_b200 import tila_api

    if not hasattr(tila.bench, "_pin_malloc_threshold"):  # reference defect, SURVEY.md §8c
        tila.bench._pin_malloc_threshold = tila.bench._pin_allocator
    for name in PATCHED:
        setattr(tila, name, getattr(tila_api, name))
        if hasattr(tila.verify, name):
            setattr(tila.verify, name, getattr(tila_api, name))
    config.addinivalue_line("markers", "gpu_adapter: reference test run against the GPU adapter")
