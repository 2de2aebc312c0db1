"""f1 depth-prior precompute: oracle vs the reference golden (CPU) and the
device kernels vs the golden + the reference's own known-answer cases (GPU).

Reference: voxsplat depth_prior.py:85-214, tests/test_depth_prior.py.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_view, load_golden

import oracle.depth_prior as odp


@pytest.fixture(scope="module")
def gold():
    return load_golden("depth_prior")


def _ocam(d, p):
    fx, fy, cx, cy = d[f"{p}_intr"]
    w, h = d[f"{p}_size"]
    return odp.Cam(d[f"{p}_r"], d[f"{p}_t"], fx, fy, cx, cy, w, h)


# ------------------------------------------------------------------ oracle (CPU)

def test_oracle_fit_align_match_reference(gold):
    for i in range(3):
        s, b, n, k = odp.fit(gold[f"raw{i}"], _ocam(gold, f"v{i}"), gold["points"])
        ref = gold[f"fit{i}"]
        assert s == pytest.approx(ref[0], rel=1e-12)
        assert b == pytest.approx(ref[1], rel=1e-12, abs=1e-12)
        assert (n, k) == (int(ref[2]), int(ref[3]))
        vals, ok = odp.align(gold[f"raw{i}"], s, b)
        np.testing.assert_array_equal(ok, gold[f"aligned{i}_valid"])
        np.testing.assert_allclose(vals, gold[f"aligned{i}_values"], rtol=1e-13, atol=0)


def test_oracle_round_trip_and_enhance_match_reference(gold):
    cams = [_ocam(gold, f"v{i}") for i in range(3)]
    al = [(gold[f"aligned{i}_values"], gold[f"aligned{i}_valid"]) for i in range(3)]
    e = odp.round_trip(al[0][0], al[0][1], cams[0], al[1][0], al[1][1], cams[1])
    np.testing.assert_array_equal(np.isfinite(e), np.isfinite(gold["err01"]))
    f = np.isfinite(e)
    np.testing.assert_allclose(e[f], gold["err01"][f], rtol=0, atol=1e-12)
    nb = odp.neighbours(cams, 0)
    assert nb == list(gold["neighbors0"])
    vals, ok, emin = odp.enhance(al[0][0], al[0][1], cams[0],
                                 [(al[j][0], al[j][1], cams[j]) for j in nb], 1.0)
    np.testing.assert_array_equal(ok, gold["enh0_valid"])
    np.testing.assert_array_equal(vals, gold["enh0_values"])
    f = np.isfinite(emin)
    np.testing.assert_array_equal(f, np.isfinite(gold["enh0_min_roundtrip"]))
    np.testing.assert_allclose(emin[f], gold["enh0_min_roundtrip"][f], rtol=0, atol=1e-12)


def test_fixture_stripe_rejected(gold):
    # the corrupted rows of view 0 are measured and rejected by the reference
    emin, ok = gold["enh0_min_roundtrip"], gold["enh0_valid"]
    stripe = np.zeros(ok.shape, bool)
    stripe[30:34, :] = True
    measured = np.isfinite(emin)
    assert not ok[stripe & measured].any()
    assert ok[~stripe & measured].mean() > 0.9


# ------------------------------------------------------------------ device (GPU)

def _views(gold):
    return [golden_view(gold, f"v{i}", i) for i in range(3)]


@pytest.mark.gpu
def test_device_fit_align_match_reference(gold):
    from paper_2503_23044_b200 import depth_prior as dp
    views = _views(gold)
    for i in range(3):
        fit = dp.fit_scale_shift(gold[f"raw{i}"], views[i], gold["points"])
        ref = gold[f"fit{i}"]
        assert fit.scale == pytest.approx(ref[0], rel=1e-10)
        assert fit.shift == pytest.approx(ref[1], rel=1e-9, abs=1e-10)
        assert (fit.samples, fit.inliers) == (int(ref[2]), int(ref[3]))
        al = dp.apply_scale_shift(gold[f"raw{i}"], fit)
        np.testing.assert_array_equal(al.valid.cpu().numpy(), gold[f"aligned{i}_valid"])
        np.testing.assert_allclose(al.values.cpu().numpy(), gold[f"aligned{i}_values"],
                                   rtol=1e-10, atol=1e-12)


@pytest.mark.gpu
def test_device_round_trip_and_enhance_match_reference(gold):
    from paper_2503_23044_b200 import depth_prior as dp
    views = _views(gold)
    al = [dp.AlignedDepthMap(gold[f"aligned{i}_values"], gold[f"aligned{i}_valid"])
          for i in range(3)]
    e = dp.reprojection_error(al[0], views[0], al[1], views[1]).cpu().numpy()
    np.testing.assert_array_equal(np.isfinite(e), np.isfinite(gold["err01"]))
    f = np.isfinite(e)
    np.testing.assert_allclose(e[f], gold["err01"][f], rtol=0, atol=1e-10)
    nb = dp.select_neighbors(views, 0)
    assert nb == list(gold["neighbors0"])
    enh = dp.enhance(al[0], views[0], [(al[j], views[j]) for j in nb], tau=1.0)
    np.testing.assert_array_equal(enh.valid.cpu().numpy(), gold["enh0_valid"])
    np.testing.assert_array_equal(enh.values.cpu().numpy(), gold["enh0_values"])
    m = enh.min_roundtrip.cpu().numpy()
    f = np.isfinite(m)
    np.testing.assert_array_equal(f, np.isfinite(gold["enh0_min_roundtrip"]))
    np.testing.assert_allclose(m[f], gold["enh0_min_roundtrip"][f], rtol=0, atol=1e-10)
    assert enh.tau == 1.0


@pytest.mark.gpu
def test_device_prepare_depth_priors_equals_stepwise(gold):
    from paper_2503_23044_b200 import depth_prior as dp
    views = _views(gold)
    out = dp.prepare_depth_priors(views, [gold[f"raw{i}"] for i in range(3)], gold["points"])
    np.testing.assert_array_equal(out[0].valid.cpu().numpy(), gold["enh0_valid"])


# Known-answer cases of the reference suite (test_depth_prior.py), on device.

def _identity_view(w, h, f):
    from paper_2503_23044_b200.geometry import CameraView
    return CameraView(0, w, h, f, f, (w - 1) / 2.0, (h - 1) / 2.0, np.eye(3), np.zeros(3))


def _look_view(view_id, w, h, eye, target, f):
    from paper_2503_23044_b200.geometry import CameraView, look_at
    r, t = look_at(np.asarray(eye, float), np.asarray(target, float))
    return CameraView(view_id, w, h, f, f, (w - 1) / 2.0, (h - 1) / 2.0, r, t)


@pytest.mark.gpu
def test_device_fit_planted_affine_and_mad_refit():
    from paper_2503_23044_b200 import depth_prior as dp
    rng = np.random.default_rng(2)
    view = _identity_view(48, 48, 50.0)
    uu, vv = np.meshgrid(np.arange(48.0), np.arange(48.0))
    metric = 1.5 + 0.06 * uu + 0.06 * vv
    s_true, b_true = 0.7, 0.35
    raw = (metric - b_true) / s_true
    raw[40:46, :] *= 1.35
    u = np.concatenate([rng.uniform(2, 45, 110), rng.uniform(2, 45, 8)])
    v = np.concatenate([rng.uniform(2, 38, 110), rng.uniform(41, 44, 8)])
    z = 1.5 + 0.06 * u + 0.06 * v
    pts = np.stack([(u - view.cx) / view.fx * z, (v - view.cy) / view.fy * z, z], axis=-1)
    fit = dp.fit_scale_shift(raw, view, pts)
    assert fit.samples == 118 and fit.inliers <= 110
    assert fit.scale == pytest.approx(s_true, rel=1e-9)
    assert fit.shift == pytest.approx(b_true, rel=1e-6)


@pytest.mark.gpu
def test_device_fit_errors():
    from paper_2503_23044_b200 import depth_prior as dp
    from paper_2503_23044_b200.errors import DegenerateFit, InsufficientData, InvalidInput
    view = _identity_view(16, 16, 20.0)
    with pytest.raises(InsufficientData):
        dp.fit_scale_shift(np.ones((16, 16)), view, np.zeros((3, 3)) + [0, 0, 2.0])
    rng = np.random.default_rng(3)
    u = rng.uniform(2, 13, 20)
    v = rng.uniform(2, 13, 20)
    pts = np.stack([(u - view.cx) / view.fx * 2.0, (v - view.cy) / view.fy * 2.0,
                    np.full(20, 2.0)], -1)
    with pytest.raises(DegenerateFit):
        dp.fit_scale_shift(np.ones((16, 16)), view, pts)
    with pytest.raises(InvalidInput):
        dp.fit_scale_shift(np.ones(16), view, pts)


@pytest.mark.gpu
def test_device_apply_scale_shift_masks_nonpositive():
    from paper_2503_23044_b200 import depth_prior as dp
    fit = dp.ScaleShiftFit(scale=2.0, shift=-1.0, samples=10, inliers=10)
    al = dp.apply_scale_shift(np.array([[1.0, 0.2], [0.0, np.nan]]), fit)
    np.testing.assert_allclose(al.values.cpu().numpy(), [[1.0, 0.0], [0.0, 0.0]])
    np.testing.assert_array_equal(al.valid.cpu().numpy(), [[True, False], [False, False]])


@pytest.mark.gpu
def test_device_round_trip_zero_inf_and_tau():
    from paper_2503_23044_b200 import depth_prior as dp
    from paper_2503_23044_b200.errors import InvalidInput
    va = _identity_view(40, 40, 45.0)
    da = np.full((40, 40), 2.0)
    vb = _look_view(1, 40, 40, (0.3, 0.1, -0.2), (0.3, 0.1, 5.0), 45.0)
    a = dp.AlignedDepthMap(da, np.ones_like(da, bool))
    b = dp.AlignedDepthMap(np.full((40, 40), 2.2), np.ones((40, 40), bool))
    err = dp.reprojection_error(a, va, b, vb).cpu().numpy()
    f = np.isfinite(err)
    assert f.mean() > 0.5 and float(err[f].max()) < 1e-9
    behind = _look_view(1, 40, 40, (0, 0, 10.0), (0, 0, 20.0), 45.0)
    err = dp.reprojection_error(a, va, dp.AlignedDepthMap(da.copy(), np.ones_like(da, bool)),
                                behind).cpu().numpy()
    assert np.all(np.isinf(err))
    with pytest.raises(InvalidInput):
        dp.enhance(a, va, [(b, vb)], tau=0.0)
