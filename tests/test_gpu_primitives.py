"""Device primitives behind the path against torch on the same inputs:
ordered stream compaction (vsx_select, the culling step's active list) and
the z-sort front (float32 proxies, identity values and digit histograms in
one kernel) through vsx_sort_splats_z."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 7, 2047, 2048, 2049, 200_053, 1_000_003])
@pytest.mark.parametrize("density", [0.0, 0.3, 1.0])
def test_select_is_flatnonzero(n, density):
    from paper_2503_23044_b200 import device as D
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    g = torch.Generator(device="cuda").manual_seed(n)
    flags = (torch.rand(n, device="cuda", generator=g) < density).to(torch.uint8)
    idx, cnt = D.select_async(flags)
    ref = torch.nonzero(flags).flatten().int()
    assert int(cnt.item()) == ref.numel()
    assert torch.equal(idx[: ref.numel()].int(), ref)


def test_select_unaligned_flags():
    """A flags view that starts at an odd byte takes the scalar load path."""
    from paper_2503_23044_b200 import device as D
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    base = (torch.arange(10_001, device="cuda") % 3 == 0).to(torch.uint8)
    flags = base[1:]
    idx, cnt = D.select_async(flags)
    ref = torch.nonzero(flags).flatten().int()
    assert int(cnt.item()) == ref.numel() and torch.equal(idx[: ref.numel()].int(), ref)


@pytest.mark.parametrize("n", [5, 4095, 620_011])
def test_sort_splats_z_is_stable_argsort(n):
    from paper_2503_23044_b200 import device as D
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    rng = np.random.default_rng(n)
    z = np.round(rng.uniform(0.5, 900.0, n), 4)          # exact ties included
    z[rng.integers(0, n, max(1, n // 50))] = np.inf        # culled entries sort last
    key = torch.as_tensor(z).cuda().view(torch.int64)
    key = torch.where(torch.as_tensor(np.isinf(z)).cuda(), torch.full_like(key, -1), key)
    order = D.sort_splats_z(key, n).cpu().numpy()
    ref = np.argsort(np.where(np.isinf(z), np.inf, z), kind="stable")
    np.testing.assert_array_equal(order[:n], ref)
