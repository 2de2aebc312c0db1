"""f4 TSDF integration on the device vs the reference (fusion.py:102-133)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_view, load_golden


@pytest.mark.gpu
def test_device_tsdf_integrate_matches_reference():
    from paper_2503_23044_b200.fusion import TsdfVolume
    g = load_golden("fusion")
    d = load_golden("depth_prior")
    vol = TsdfVolume.from_bounds([-3.0, -2.0, -0.5], [3.0, 3.0, 0.5], 0.1, 0.3)
    assert vol.dims == tuple(int(x) for x in g["dims"])
    touched = [vol.integrate(d[f"aligned{i}_values"], d[f"aligned{i}_valid"],
                             golden_view(d, f"v{i}", i)) for i in range(3)]
    assert touched == g["touched"].tolist()
    tsdf, weight = (x.reshape(-1) for x in vol.grids())
    np.testing.assert_array_equal(weight, g["weight"])
    np.testing.assert_allclose(tsdf, g["tsdf"], rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_device_tsdf_validation():
    from paper_2503_23044_b200.errors import InvalidInput, ResourceError
    from paper_2503_23044_b200.fusion import TsdfVolume
    with pytest.raises(InvalidInput):
        TsdfVolume([0, 0, 0], (1, 4, 4), 0.1, 0.3)
    with pytest.raises(InvalidInput):
        TsdfVolume([0, 0, 0], (4, 4, 4), 0.1, 0.05)
    with pytest.raises(ResourceError):
        TsdfVolume.from_bounds([0, 0, 0], [10, 10, 10], 0.01, 0.05, budget=1000)
    v = TsdfVolume.from_bounds([0, 0, 0], [10, 10, 10], 0.01, 0.05, budget=1000,
                               auto_coarsen=True)
    assert int(np.prod(v.dims)) <= 1000 and v.observed_fraction == 0.0
