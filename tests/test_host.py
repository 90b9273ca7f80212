"""Host-side logic of the torch and tila-mirror APIs that runs before any
device work: argument validation mirrors the reference's ValueError cases
(pkg/src/tila/reference.py:42-74, kernel.py:68-70) and CPU tensors are refused
(there is no CPU path). CPU only."""

import numpy as np
import pytest
import torch

import paper_2401_04658_b200 as la2
from paper_2401_04658_b200 import tila_api


def test_decay_validation():
    t = la2.decay_tensor([0.5, 1.0], 2, torch.device("cpu"))
    assert t.dtype == torch.float32 and t.tolist() == [0.5, 1.0]
    assert la2.decay_tensor(0.9, 3, torch.device("cpu")).shape == (3,)
    for bad in (0.0, -0.1, 1.5, float("nan")):
        with pytest.raises(ValueError):
            la2.decay_tensor([bad, 0.5], 2, torch.device("cpu"))
    with pytest.raises(ValueError):
        la2.decay_tensor([0.5, 0.5, 0.5], 2, torch.device("cpu"))


def test_cpu_tensors_refused():
    q = torch.zeros(1, 2, 8, 64)
    with pytest.raises(ValueError, match="CUDA"):
        la2.lightning_attn2(q, q, q, [0.9, 0.9])
    # every entry point refuses host tensors before any device work (a host pointer
    # reaching a kernel would fault): decode, multi-token decode, recurrence, Norm(.)
    st = torch.zeros(1, 2, 64, 64)
    with pytest.raises(ValueError, match="CUDA"):
        la2.decode_step(q[:, :, 0], q[:, :, 0], q[:, :, 0], [0.9, 0.9], st)
    with pytest.raises(ValueError, match="CUDA"):
        la2.decode_tokens(q, q, q, [0.9, 0.9], st)
    with pytest.raises(ValueError, match="CUDA"):
        la2.recurrent_forward(q, q, q, [0.9, 0.9])
    with pytest.raises(ValueError, match="CUDA"):
        la2.ops.rmsnorm_forward(q)
    with pytest.raises(ValueError, match="CUDA"):
        la2.ops.rmsnorm_backward(q, q, torch.zeros(1, 2, 8))


def test_shape_errors():
    q = torch.zeros(1, 2, 8, 64)
    with pytest.raises(ValueError):
        la2.la2_forward(q, torch.zeros(1, 2, 8, 32), q, 0.9)
    with pytest.raises(ValueError):
        la2.la2_forward(q, q, torch.zeros(1, 2, 9, 64), 0.9)
    with pytest.raises(ValueError):
        la2.la2_forward(q[0], q[0], q[0], 0.9)


def test_tila_api_validation_matches_reference():
    with pytest.raises(ValueError):
        tila_api.tiled_forward(np.ones((2, 3)), np.ones((2, 4)), np.ones((2, 3)), 0.5, 4)
    with pytest.raises(ValueError):
        tila_api.tiled_forward(np.ones((2, 3)), np.ones((2, 3)), np.ones((3, 3)), 0.5, 4)
    with pytest.raises(ValueError):
        tila_api.tiled_forward(np.ones((2, 3)), np.ones((2, 3)), np.ones((2, 3)), 1.5, 4)
    with pytest.raises(ValueError):
        tila_api.tiled_forward(np.ones((2, 3)), np.ones((2, 3)), np.ones((2, 3)), 0.5, 0)
    with pytest.raises(ValueError):
        tila_api.tiled_backward(np.ones((2, 2)), np.ones((2, 2)), np.ones((2, 3)), np.ones((2, 2)), 0.9, 4)
    with pytest.raises(ValueError):
        tila_api.chunked_forward(np.ones((8, 4)), np.ones((8, 4)), np.ones((8, 4)), 0.9, 4,
                                 tila_api.KvState.fresh(3, 4))
    with pytest.raises(ValueError, match="head 1"):
        good = (np.ones((8, 4)), np.ones((8, 4)), np.ones((8, 4)), 0.9)
        bad = (np.ones((8, 4)), np.ones((8, 5)), np.ones((8, 4)), 0.9)
        tila_api.batched_forward([good, bad], 4)
    with pytest.raises(ValueError):
        tila_api.inference_step([1.0, 2.0], [1.0, 2.0, 3.0], [1.0, 2.0, 3.0],
                                tila_api.KvState.fresh(3, 3), 0.9)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_tila_api_requires_gpu():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        tila_api.tiled_forward(np.ones((2, 3)), np.ones((2, 3)), np.ones((2, 3)), 0.5, 4)


def test_split_factor_policy():
    """Intra-GPU sequence split: tensor-core shapes split only when units underfill the
    GPU (chunks >= 8192 tokens, at least 4-way); SIMT shapes (fp32) split to ~4 units per SM (chunks >= 32
    tokens at d <= 64, >= 128 above; at most 64 chunks)."""
    import torch
    from paper_2401_04658_b200.ops import split_factor
    assert split_factor(8, 16, 65536, 64, 64, torch.bfloat16) == 1        # C2: 128 units
    assert split_factor(1, 16, 524288, 128, 128, torch.bfloat16) == 8     # C5 on one GPU
    assert split_factor(1, 2, 300, 64, 64, torch.bfloat16) == 1           # too short
    assert split_factor(1, 8, 8192, 64, 64, torch.bfloat16) == 1          # 2-way never pays
    assert split_factor(1, 16, 16384, 64, 64, torch.bfloat16) == 1        # chunks < 8192 tokens
    assert split_factor(1, 4, 65536, 64, 64, torch.bfloat16) == 8
    assert split_factor(1, 8, 2048, 64, 64, torch.float32) == 64          # C1 fp32 (SIMT)
    assert split_factor(1, 8, 1024, 64, 64, torch.float32) == 32          # 32-token chunks
    assert split_factor(1, 8, 2048, 128, 128, torch.float32) == 16        # d=128: >= 128 tokens
    assert split_factor(1, 1, 1 << 20, 64, 64, torch.float32) == 64       # scan limit
    assert split_factor(1, 3, 333, 4, 7, torch.float32) == 1              # odd length
    assert split_factor(64, 16, 4096, 64, 64, torch.float32) == 1         # already 1024 units
    # long few-head sequences: never more chunks than la2_state_scan combines (64)
    for shape in ((1, 1, 1 << 20, 64, 64), (1, 2, 1 << 20, 64, 64), (1, 1, 1 << 20, 128, 128),
                  (1, 2, 1 << 20, 128, 128), (1, 1, 1 << 21, 64, 64), (1, 1, 1 << 23, 128, 128)):
        g = split_factor(*shape, torch.bfloat16)
        assert 1 <= g <= 64 and shape[2] % g == 0, (shape, g)
    assert split_factor(1, 1, 1 << 21, 64, 64, torch.bfloat16) == 64


def test_gpubench_verdict_and_csv(tmp_path):
    """The GPU harness keeps the reference's classify bands, sweep rule and CSV schema
    (pkg/src/tila/bench.py:33-36, :99-108, :230-235, :301-314)."""
    from paper_2401_04658_b200 import gpubench as gb
    assert gb.CSV_HEADER == "impl,direction,n,d,dv,B,lambda,reps,median_s,us_per_token,scratch_bytes"
    assert gb.classify([2.0, 2.1, 1.9]) == "linear-like"
    assert gb.classify([4.0, 4.1]) == "quadratic-like"
    assert gb.classify([2.0, 4.0]) == "inconclusive"
    assert gb.classify([]) == "inconclusive"
    assert gb.classify([float("nan")]) == "inconclusive"
    with pytest.raises(ValueError):
        gb._check_n_list([128, 256, 512])
    with pytest.raises(ValueError):
        gb._check_n_list([128, 256, 500, 1000])
    rec = gb.BenchRecord("tiled", "fwd+bwd", 1024, 64, 64, 64, 0.9, 5, 1e-4, 0.1, 0)
    p = tmp_path / "x.csv"
    gb.emit_csv([rec], p)
    lines = p.read_text().splitlines()
    assert lines[0] == gb.CSV_HEADER
    assert lines[1] == "tiled,fwd+bwd,1024,64,64,64,0.90000000000000002,5,0.0001,0.10000000000000001,0"
    with pytest.raises(ValueError):
        gb.emit_csv([], p)
    # criterion 5 of the reference's acceptance suite (test_acceptance.py:51-62)
    assert gb.ACCEPTANCE_N == (8192, 16384, 32768, 65536) and gb.ACCEPTANCE_SPREAD == 1.5
    gb._check_n_list(gb.ACCEPTANCE_N)


def test_cli_usage_errors_exit_2():
    """CLI parity with the reference (pkg/src/tila/cli.py): bad sweeps are usage errors."""
    from paper_2401_04658_b200 import cli
    for argv in (["bench", "--impls", "tiled", "--lens", "128,256,512", "--dim", "64", "--block", "64"],
                 ["bench", "--impls", "tiled", "--lens", "128,256,500,1000", "--dim", "64", "--block", "64"],
                 ["bench", "--impls", "oracle", "--lens", "128,256,512,1024", "--dim", "64", "--block", "64"],
                 ["nope"]):
        with pytest.raises(SystemExit) as e:
            cli.main(argv)
        assert e.value.code == 2
    args = cli.build_parser().parse_args(["stream-demo", "--dim", "64", "--chunk", "100", "--chunks", "3"])
    assert args.lam == cli.BENCH_LAMBDA


def test_bench_roofline_traffic_source():
    """bench.py's per-launch roofline.traffic comes from the committed ncu summary: DRAM
    bytes per token-head of each launch of one d=64 step, each close to its compulsory
    bytes."""
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import bench
    per = bench.load_ncu_bytes(64)
    # forward F storing the per-block states (4 tensors + half a tensor of states), then the
    # dQ/dK/dV triple (reads K, Q, dO, V and the states once; writes dQ, dK, dV)
    assert per is not None and set(per) == {"forward", "backward"}, per
    for role, alg in (("forward", 512 + 64), ("backward", 7 * 128 + 64)):
        assert 0.9 * alg <= per[role] <= 1.1 * alg, (role, per)


def test_bench_launch_roles():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    recs = [{"kernel": "a", "grid": 1, "cluster": 1, "ms": 1.0}, {"kernel": "b", "grid": 2, "cluster": 2, "ms": 3.0},
            {"kernel": "a", "grid": 1, "cluster": 1, "ms": 2.0}, {"kernel": "b", "grid": 2, "cluster": 2, "ms": 5.0}]
    r = bench.launch_roles(recs, ["dq", "dkdv"])
    assert r["dq"]["ms"] == 1.5 and r["dkdv"]["ms"] == 4.0 and r["dkdv"]["kernel"] == "b"
    assert bench.launch_roles(recs[:3], ["dq", "dkdv"]) == {}


def test_cuda_decay_check_cache(monkeypatch):
    """la2_check_decay runs once per (tensor, version): a new tensor at a recycled address,
    or an in-place change, is checked again (host logic; the C call is stubbed)."""
    import torch
    from paper_2401_04658_b200 import ops
    calls = []
    monkeypatch.setattr(ops._lib, "call", lambda name, *a: calls.append(name))
    monkeypatch.setattr(ops, "_stream", lambda dev: 0)
    monkeypatch.setattr(torch.cuda, "is_current_stream_capturing", lambda: False)
    t = torch.tensor([0.5, 0.9])
    ops._check_cuda_decay(t)
    ops._check_cuda_decay(t)
    assert calls == ["la2_check_decay"]
    t.mul_(1.0)  # bumps the version
    ops._check_cuda_decay(t)
    assert len(calls) == 2
    u = torch.tensor([0.5, 0.9])  # another tensor object: checked
    ops._check_cuda_decay(u)
    assert len(calls) == 3
    # a derived vector is cached under the caller's tensor
    w = torch.tensor([0.5, 0.9], dtype=torch.float64)
    ops._check_cuda_decay(w.float(), w)
    ops._check_cuda_decay(w.float(), w)
    assert len(calls) == 4


def test_bench_reference_arm_contract():
    """bench.py --impl reference: rank 0 times the reference's own CPU implementation and
    prints the contract's JSON line (impl, metric, value, cpu_baseline, e2e with zero
    copy bytes); under torchrun the other ranks exit 0 without work or output."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    base = [sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
            "--batch", "1", "--heads", "2", "--seq-len", "512", "--cpu-sample-heads", "2"]
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run(base, cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "", (r.stdout, r.stderr[-2000:])
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run(base, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_missing_library_fails_loudly():
    """Without the built library the ops raise ImportError ("no CPU fallback") instead of
    computing anything on the host."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = ("import paper_2401_04658_b200 as la2\n"
            "from paper_2401_04658_b200 import _lib\n"
            "try:\n"
            "    _lib.load()\n"
            "except ImportError as e:\n"
            "    print('ImportError:', e)\n")
    env = dict(os.environ, LA2_LIB=str(root / "does_not_exist" / "libla2.so"))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ImportError" in r.stdout and "no CPU fallback" in r.stdout, (r.stdout, r.stderr)
