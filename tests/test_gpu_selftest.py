"""tcgen05 operand-layout self-test: one GEMM per (M, N, K, A-major, B-major)
through the same SW128 descriptors the Lightning-2 kernel uses."""

import itertools

import pytest
import torch

from paper_2401_04658_b200 import _lib

pytestmark = pytest.mark.gpu


CASES = list(itertools.product((64, 128), (64, 128), (64, 128), (0, 1), (0, 1)))
# a_mn == 2: A operand read from TMEM (tcgen05.mma ... [a_tmem]); for M = 64 the A rows
# sit in lanes 0-15 of each 32-lane quarter, like the M = 64 accumulator layout
CASES += list(itertools.product((64, 128), (64, 128), (64, 128), (2,), (0, 1)))


@pytest.mark.parametrize("M,N,K,a_mn,b_mn", CASES)
def test_umma_layouts(M, N, K, a_mn, b_mn):
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K + 2 * a_mn + b_mn)
    A = (torch.rand(M, K, generator=g) * 2 - 1).bfloat16().float()
    B = (torch.rand(K, N, generator=g) * 2 - 1).bfloat16().float()
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.full((M, N), float("nan"), device="cuda")
    _lib.call_dev("la2_selftest_umma", Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), M, N, K, a_mn, b_mn,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = A.double() @ B.double()
    err = (D.cpu().double() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
