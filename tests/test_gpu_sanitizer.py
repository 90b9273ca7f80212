"""compute-sanitizer over one small fwd+bwd step of the tcgen05 kernels (memcheck,
racecheck, synccheck, initcheck), replay and stored-state backward: no out-of-bounds / uninitialised global accesses, no
shared-memory hazards, no illegal barrier use."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool,shape", [
    ("memcheck", "2,3,1000,64"),
    ("memcheck", "1,5,777,128"),
    ("memcheck", "4,40,1000,64"),   # more units than SMs: persistent stream-K ranges
    ("memcheck", "2,40,700,128"),
    ("racecheck", "1,3,700,64"),
    ("synccheck", "1,3,700,64"),
    ("initcheck", "1,3,700,128"),
    # the d = 64 stored-state triple (forward storing the states, shared dK/dV recurrence
    # with st.async operand exchange, stateless dQ CTA), also across persistent ranges
    ("memcheck", "1,3,700,64,s"),
    ("memcheck", "4,40,1000,64,s"),
    ("racecheck", "1,3,700,64,s"),
    ("synccheck", "1,3,700,64,s"),
    # the fused Norm(.) epilogue (the two row warps of a quarter exchange row sums in smem)
    ("racecheck", "1,3,700,64,n"),
    ("memcheck", "2,40,700,64,n"),
    # multi-token decode (register-resident state slices, chunked q/k staging, next-chunk
    # prefetch): a partial last chunk, two column slices per head at d = 128
    ("memcheck", "2,3,19,128,t"),
    ("racecheck", "2,3,19,128,t"),
    ("initcheck", "1,2,11,64,t"),
    # fp32 on the register-tiled SIMT kernels: split path (chunk states, scans) and raw passes,
    # a partial last block and a width that is not a multiple of 4
    ("memcheck", "1,3,1000,64,f"),
    ("racecheck", "1,2,300,20,f"),
    ("initcheck", "1,2,300,20,f"),
])
def test_sanitizer_clean(tool, shape):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "3", "--print-limit", "10",
           sys.executable, os.path.join(ROOT, "tools", "one_step.py"), shape]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert ("ERROR SUMMARY: 0 errors" in out) or ("0 hazards" in out), out[-4000:]
