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
