"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact: culling masks, radix-sort order, tile lists. Float: images within
1e-4 absolute, gradients within 1e-3 relative (+ a small absolute floor),
on guard-margin pixels where the reference tests apply the same exclusion
(helpers.py:129-137 of the reference suite).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from conftest import golden_view, golden_scene
from gpu_util import f32r, oracle_splats, records_from, rel_close, splat_arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2503_23044_b200 import _lib
    _lib.load()


# ------------------------------------------------------------------ primitives

@pytest.mark.parametrize("n", [1, 5, 4096, 4097, 70001])
def test_radix_sort_u64_is_stable(n):
    from paper_2503_23044_b200 import device as D
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 50, size=n).astype(np.uint64) * np.uint64(0x10000000001) + \
        np.uint64(0x3F00000000000000)
    k = torch.as_tensor(keys.view(np.int64)).cuda()
    v = torch.arange(n, dtype=torch.int32, device="cuda")
    ko, vo = D.sort_pairs_u64(k, v, n)
    expect = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(vo.cpu().numpy(), expect)
    np.testing.assert_array_equal(ko.cpu().numpy().view(np.uint64), keys[expect])


@pytest.mark.parametrize("n", [1, 2048, 2049, 3_000_001])
def test_exclusive_scan(n):
    from paper_2503_23044_b200 import device as D
    rng = np.random.default_rng(1)
    c = rng.integers(0, 7, size=n).astype(np.int32)
    out = D.exclusive_scan(torch.as_tensor(c).cuda(), n).cpu().numpy()
    np.testing.assert_array_equal(out[:-1], np.concatenate([[0], np.cumsum(c)[:-1]]))
    assert out[-1] == c.sum()


# ------------------------------------------------------------------ K1 culling

@pytest.mark.parametrize("tag", ["far", "near"])
def test_cull_bitexact_vs_reference_golden(scene_small, tag):
    from paper_2503_23044_b200.scene import active_mask
    scene = golden_scene(scene_small)
    view = golden_view(scene_small, tag)
    for k in range(scene.lod_count):
        np.testing.assert_array_equal(active_mask(scene, k, view), scene_small[f"{tag}_mask{k}"])


def test_cull_bitexact_random_scene():
    from paper_2503_23044_b200.device import DeviceScene
    from paper_2503_23044_b200.geometry import make_view
    from paper_2503_23044_b200.scene import SparsePoints, build_hierarchy
    rng = np.random.default_rng(11)
    scene = build_hierarchy(SparsePoints(rng.uniform(-4, 4, size=(60000, 3))), 0.4, 4,
                            offsets_per_voxel=2, seed=1)
    ds = DeviceScene(scene)
    for i in range(6):
        eye = rng.uniform(-6, 6, 3)
        view = make_view(i, 320, 200, eye, rng.uniform(-1, 1, 3), fov_deg=70)
        mask = ds.cull(view).cpu().numpy().astype(bool)
        ref = oracle.cull(scene.flat_centers(), scene.flat_levels(), scene.lod_count,
                          scene.lod_ref_distance, 0, oracle.Cam.of(view))
        np.testing.assert_array_equal(mask, ref)


# ------------------------------------------------------------------ K2 decode

def _decode_pair(d, tag, n=2):
    """Device decode vs the oracle on float32-rounded parameters."""
    from paper_2503_23044_b200.decoder import AnchorState, DecoderParams, decode_active
    scene = golden_scene(d)
    view = golden_view(d, tag)
    weights = {k[2:]: d[k] for k in d if k.startswith("w_")}
    params = DecoderParams.from_arrays(n, weights)
    state = AnchorState.from_scene(scene)
    batch = decode_active(params, scene, view, state=state)
    centers, levels = scene.flat_centers(), scene.flat_levels()
    cam = oracle.Cam.of(view)
    act = np.flatnonzero(oracle.cull(centers, levels, scene.lod_count, scene.lod_ref_distance,
                                     0, cam))
    w64 = {k: torch.tensor(f32r(v)) for k, v in weights.items()}
    emb = torch.tensor(f32r(scene.flat("embeddings")))[act]
    ls = torch.tensor(f32r(np.log(scene.flat("scales"))))[act]
    off = torch.tensor(f32r(scene.flat("offsets")))[act]
    dec = oracle.flatten_decoded(oracle.decode(w64, centers[act], emb, torch.exp(ls), off,
                                               cam.center, scene.lod_ref_distance,
                                               3 * scene.base_voxel_size, n))
    return batch, dec, act, scene, view


@pytest.mark.parametrize("tag", ["far", "near"])
def test_decode_matches_oracle(scene_small, tag):
    batch, dec, act, _, _ = _decode_pair(scene_small, tag)
    np.testing.assert_array_equal(batch.gid, (act[:, None] * 2 + np.arange(2)).reshape(-1))
    np.testing.assert_allclose(batch.means.cpu().numpy(), dec["means"].numpy(), rtol=1e-14,
                               atol=1e-15)
    for k, got in (("opacities", batch.opacities), ("colors", batch.colors),
                   ("scales", batch.scales), ("quats", batch.quats), ("normals", batch.normals)):
        np.testing.assert_allclose(got.cpu().numpy(), dec[k].numpy(), rtol=2e-5, atol=2e-6,
                                   err_msg=k)


# ------------------------------------------------------------------ K3 projection + sort

@pytest.mark.parametrize("tag", ["far", "near"])
def test_project_order_and_values_match_oracle(scene_small, tag):
    from paper_2503_23044_b200.renderer import project_splats
    batch, _, act, _, view = _decode_pair(scene_small, tag)
    splats = project_splats(batch, view)
    # oracle on exactly the device's decoded inputs
    g = {"means": torch.tensor(batch.means.cpu().numpy()),
         **{k: torch.tensor(getattr(batch, k).cpu().numpy().astype(np.float64))
            for k in ("opacities", "colors", "scales", "quats", "normals")}}
    P = oracle.project(g, batch.gid, oracle.Cam.of(view))
    np.testing.assert_array_equal(splats.gid, P["gid"])
    np.testing.assert_array_equal(splats.zkey, P["zkey"])
    np.testing.assert_allclose(splats.mean2d.cpu().numpy(), P["mean2d"].numpy(), rtol=0,
                               atol=1e-9)
    np.testing.assert_allclose(splats.radius, P["radius"], rtol=1e-12)
    for k in ("conic", "color", "normal_cam", "plane_d", "opacity"):
        np.testing.assert_allclose(getattr(splats, k).cpu().numpy(), P[k].numpy(), rtol=1e-6,
                                   atol=1e-7, err_msg=k)


# ------------------------------------------------------------------ K4 binning

@pytest.mark.parametrize("tag", ["far", "near"])
def test_bin_lists_bitexact_vs_reference(scene_small, tag):
    from paper_2503_23044_b200 import device as D
    d = scene_small
    view = golden_view(d, tag)
    spl = {k: d[f"{tag}_spl_{k}"] for k in ("mean2d", "conic", "color", "opacity",
                                             "normal_cam", "plane_d", "radius", "zkey")}
    B = D.bin_tiles(records_from(spl), view.width, view.height)
    np.testing.assert_array_equal(B.tile_offsets.cpu().numpy(), d[f"{tag}_tile_off"])
    np.testing.assert_array_equal(B.tile_list.cpu().numpy(), d[f"{tag}_tile_list"])


def test_bin_lists_bitexact_random_large():
    from paper_2503_23044_b200 import device as D
    rng = np.random.default_rng(5)
    n, W, H = 200000, 1920, 1080
    spl = {"mean2d": np.stack([rng.uniform(-80, W + 80, n), rng.uniform(-80, H + 80, n)], -1),
           "radius": np.exp(rng.uniform(np.log(0.5), np.log(120.0), n)),
           "conic": np.ones((n, 3)), "color": np.zeros((n, 3)), "opacity": np.ones(n),
           "normal_cam": np.zeros((n, 3)), "plane_d": np.zeros(n)}
    # put some boxes exactly on tile boundaries
    spl["mean2d"][:1000, 0] = np.round(spl["mean2d"][:1000, 0] / 16) * 16 + spl["radius"][:1000]
    B = D.bin_tiles(records_from(spl), W, H)
    off, lst = oracle.bin_tiles(spl["mean2d"], spl["radius"], W, H)
    np.testing.assert_array_equal(B.tile_offsets.cpu().numpy(), off)
    np.testing.assert_array_equal(B.tile_list.cpu().numpy(), lst)


# ------------------------------------------------------------------ K5 compositing

@pytest.mark.parametrize("tag", ["far", "near"])
def test_raster_forward_within_1e4_of_reference(scene_small, tag):
    from paper_2503_23044_b200 import device as D
    d = scene_small
    view = golden_view(d, tag)
    spl = {k: d[f"{tag}_spl_{k}"] for k in ("mean2d", "conic", "color", "opacity",
                                             "normal_cam", "plane_d", "radius", "zkey")}
    P = records_from(spl)
    R = D.raster_forward(P, D.bin_tiles(P, view.width, view.height), view)
    for k, got in (("rgb", R.rgb), ("alpha", R.alpha), ("raw_normal", R.raw_normal)):
        err = np.abs(got.cpu().numpy() - d[f"{tag}_img_{k}"]).max()
        assert err <= 1e-4, (k, err)
    valid = d[f"{tag}_img_valid"]
    np.testing.assert_array_equal(R.valid.cpu().numpy().astype(bool), valid)
    derr = np.abs(R.depth.cpu().numpy() - d[f"{tag}_img_depth"])[valid].max()
    assert derr <= 1e-4, derr
    nerr = np.abs(R.normal.cpu().numpy() - d[f"{tag}_img_normal"]).max()
    assert nerr <= 1e-4, nerr


@pytest.mark.parametrize("case", [0, 1])
def test_render_gaussians_forward_and_gradients_vs_reference(raster_leaf, case):
    """Leaf gaussians -> project -> composite -> backward (K3/K5/K6/K7) vs golden."""
    from paper_2503_23044_b200.renderer import (rasterize_backward, rasterize_view,
                                                make_leaf_gaussians, project_splats)
    d, p = raster_leaf, f"c{case}"
    view = golden_view(d, p)
    batch = make_leaf_gaussians(d[f"{p}_means"], d[f"{p}_opacities"], d[f"{p}_colors"],
                                d[f"{p}_scales"], d[f"{p}_quats"], requires_grad=True)
    splats = project_splats(batch, view)
    np.testing.assert_array_equal(splats.gid, d[f"{p}_spl_gid"])
    targets, _ = rasterize_view(splats, view)
    for k in ("rgb", "alpha"):
        err = np.abs(getattr(targets, k).detach().cpu().numpy() - d[f"{p}_img_{k}"]).max()
        assert err <= 1e-4, (k, err)
    cot = {k: d[f"{p}_cot_{k}"] for k in ("rgb", "alpha", "depth", "normal")}
    grads = rasterize_backward(splats, {"rgb": targets.rgb, "alpha": targets.alpha,
                                        "depth": targets.depth, "normal": targets.normal}, cot)
    for k, g in grads.items():
        ref = d[f"{p}_grad_{k}"]
        scale = np.abs(ref).max()
        ok, worst, nbad = rel_close(g.detach().cpu().numpy(), ref, 1e-3, 1e-4 * scale)
        assert ok, f"{k}: {nbad} bad, worst rel {worst:.3g}"
