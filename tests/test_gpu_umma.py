"""Hardware check of the hand-written tcgen05 path (umma.cuh conventions)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("N,K", [(64, 40), (80, 64), (16, 8), (192, 40)])
def test_tcgen05_tf32_gemm_matches_fp64(N, K):
    from paper_2503_23044_b200._lib import call, ptr, stream
    rng = np.random.default_rng(N + K)
    A = rng.normal(size=(128, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    At, Bt = torch.as_tensor(A).cuda(), torch.as_tensor(B).cuda()
    for three, tol in ((0, 3e-3), (1, 2e-6)):
        D = torch.zeros((128, N), dtype=torch.float32, device="cuda")
        call("vsx_umma_selftest", ptr(At), ptr(Bt), ptr(D), N, K, three, stream())
        err = np.abs(D.cpu().numpy() - ref).max() / np.abs(ref).max()
        assert err < tol, (three, err)
