"""Pin the CPU oracle against outputs of the unmodified reference (tests/golden).

Bit-exact: culling masks, z-sort order, tile lists, the host scene builder.
Float64 outputs agree to 1e-10 absolute, gradients to 1e-8 relative (only
summation order differs from the reference).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from conftest import golden_scene, golden_view, load_golden

F64 = torch.float64


def _weights(d: dict) -> dict:
    return {k[2:]: torch.tensor(d[k]) for k in d if k.startswith("w_")}


def _flat_scene(d: dict):
    K = int(d["lod_count"])
    base = float(d["base_voxel"])
    centers = np.concatenate([d[f"grid{k}"].astype(np.float64) * (base / 2.0 ** k)
                              for k in range(K)])
    levels = np.concatenate([np.full(d[f"grid{k}"].shape[0], k) for k in range(K)])
    return centers, levels


def _grad_close(a, b, rel=1e-8, floor=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    tol = rel * np.maximum(np.abs(a), np.abs(b)) + floor
    bad = np.abs(a - b) > tol
    assert not bad.any(), f"{bad.sum()} mismatches, worst {np.abs(a - b).max():.3g}"


def test_host_build_hierarchy_reproduces_reference(scene_small):
    from paper_2503_23044_b200.scene import SparsePoints, build_hierarchy
    d = scene_small
    scene = build_hierarchy(SparsePoints(d["points"]), 0.5, 3, offsets_per_voxel=2, seed=0)
    for k in range(3):
        np.testing.assert_array_equal(scene.levels[k].grid, d[f"grid{k}"])
        np.testing.assert_array_equal(scene.levels[k].embeddings, d[f"emb{k}"])
        np.testing.assert_array_equal(scene.levels[k].offsets, d[f"off{k}"])


def test_oracle_decoder_init_reproduces_reference(scene_small):
    w = oracle.decoder_init(2, seed=0, scale_bias=float(np.log(0.1)))
    for k, t in _weights(scene_small).items():
        np.testing.assert_array_equal(w[k], t.numpy())


@pytest.mark.parametrize("tag", ["far", "near"])
def test_oracle_cull_bitexact(scene_small, tag):
    d = scene_small
    centers, levels = _flat_scene(d)
    cam = oracle.Cam.of(golden_view(d, tag))
    mask = oracle.cull(centers, levels, 3, float(d["lod_ref"]), int(d["lod_bias"]), cam)
    ref = np.concatenate([d[f"{tag}_mask{k}"] for k in range(3)])
    np.testing.assert_array_equal(mask, ref)


@pytest.mark.parametrize("tag", ["far", "near"])
def test_oracle_decode_project_bin_raster(scene_small, tag):
    d = scene_small
    centers, levels = _flat_scene(d)
    cam = oracle.Cam.of(golden_view(d, tag))
    mask = oracle.cull(centers, levels, 3, float(d["lod_ref"]), int(d["lod_bias"]), cam)
    act = np.flatnonzero(mask)
    emb = np.concatenate([d[f"emb{k}"] for k in range(3)])
    off = np.concatenate([d[f"off{k}"] for k in range(3)])
    scl = np.concatenate([d[f"scl{k}"] for k in range(3)])
    dec = oracle.flatten_decoded(oracle.decode(
        _weights(d), centers[act], torch.tensor(emb[act]), torch.tensor(scl[act]),
        torch.tensor(off[act]), cam.center, float(d["lod_ref"]), 3.0 * float(d["base_voxel"]), 2))
    for k in ("means", "opacities", "colors", "scales", "quats", "normals"):
        np.testing.assert_allclose(dec[k].numpy(), d[f"{tag}_dec_{k}"], atol=1e-12, rtol=0)
    gid = (act[:, None] * 2 + np.arange(2)).reshape(-1)
    np.testing.assert_array_equal(gid, d[f"{tag}_dec_gid"])
    P = oracle.project(dec, gid, cam)
    np.testing.assert_array_equal(P["gid"], d[f"{tag}_spl_gid"])
    np.testing.assert_array_equal(P["zkey"], d[f"{tag}_spl_zkey"])
    for k in oracle.SPLAT_KEYS:
        np.testing.assert_allclose(P[k].numpy(), d[f"{tag}_spl_{k}"], atol=1e-10, rtol=0)
    np.testing.assert_allclose(P["radius"], d[f"{tag}_spl_radius"], rtol=1e-13)
    offs, lists = oracle.bin_tiles(d[f"{tag}_spl_mean2d"], d[f"{tag}_spl_radius"],
                                   cam.width, cam.height)
    np.testing.assert_array_equal(offs, d[f"{tag}_tile_off"])
    np.testing.assert_array_equal(lists, d[f"{tag}_tile_list"])
    S = {k: torch.tensor(d[f"{tag}_spl_{k}"]) for k in oracle.SPLAT_KEYS}
    img = oracle.raster(S, offs, lists, cam)
    for k in ("rgb", "depth", "normal", "alpha", "raw_normal"):
        np.testing.assert_allclose(img[k].numpy(), d[f"{tag}_img_{k}"], atol=1e-10, rtol=0)
    np.testing.assert_array_equal(img["valid"].numpy(), d[f"{tag}_img_valid"])
    np.testing.assert_array_equal(img["counts"], d[f"{tag}_counts"])


@pytest.mark.parametrize("case", [0, 1])
def test_oracle_raster_gradients_match_reference(raster_leaf, case):
    d, p = raster_leaf, f"c{case}"
    cam = oracle.Cam.of(golden_view(d, p))
    g = oracle.leaf_gaussians(d[f"{p}_means"], d[f"{p}_opacities"], d[f"{p}_colors"],
                              d[f"{p}_scales"], d[f"{p}_quats"], requires_grad=True)
    P = oracle.project(g, np.arange(len(d[f"{p}_means"])), cam)
    np.testing.assert_array_equal(P["gid"], d[f"{p}_spl_gid"])
    for k in oracle.SPLAT_KEYS:
        np.testing.assert_allclose(P[k].detach().numpy(), d[f"{p}_spl_{k}"], atol=1e-10)
    offs, lists = oracle.bin_tiles(P["mean2d"].detach().numpy(), P["radius"],
                                   cam.width, cam.height)
    np.testing.assert_array_equal(lists, d[f"{p}_tile_list"])
    img = oracle.raster(P, offs, lists, cam)
    for k in ("rgb", "depth", "normal", "alpha"):
        np.testing.assert_allclose(img[k].detach().numpy(), d[f"{p}_img_{k}"], atol=1e-10)
    obj = sum((img[k] * torch.tensor(d[f"{p}_cot_{k}"])).sum()
              for k in ("rgb", "alpha", "depth", "normal"))
    leaves = g["leaves"]
    grads = torch.autograd.grad(obj, [leaves[k] for k in leaves])
    for k, gr in zip(leaves, grads):
        _grad_close(gr.numpy(), d[f"{p}_grad_{k}"])


def _train_state(d: dict, **cfg):
    centers, levels = _flat_scene(d)
    K = int(d["lod_count"])
    n = int(d["n"])
    w = oracle.decoder_init(n, seed=0, scale_bias=float(np.log(0.125 * float(d["base_voxel"]))))
    return oracle.OracleState.create(
        centers, levels, K, float(d["lod_ref"]), int(d["lod_bias"]), float(d["base_voxel"]), n,
        w, np.concatenate([d[f"emb{k}"] for k in range(K)]),
        np.log(np.concatenate([d[f"scl{k}"] for k in range(K)])),
        np.concatenate([d[f"off{k}"] for k in range(K)]), **cfg)


@pytest.mark.parametrize("tag", ["rgb", "depth"])
def test_oracle_train_steps_match_reference(train_small, tag):
    d = train_small
    st = _train_state(d, total_steps=8, step2_start=8 if tag == "rgb" else 0, step3_start=8)
    cams = [oracle.Cam.of(golden_view(d, f"v{i}", i)) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    priors = [(d[f"prior{i}"], d[f"pvalid{i}"]) for i in range(3)] if tag == "depth" else None
    for s in range(3):
        rep = oracle.train_step(st, cams, images, priors)
        np.testing.assert_allclose([rep["total"], rep["rgb"], rep["depth"]],
                                   d[f"{tag}_loss"][s], rtol=1e-10, atol=1e-13)
        if tag == "depth":
            assert rep["supervised_depth_px"] == d["depth_supervised"][s]
    for k, t in st.weights.items():
        np.testing.assert_allclose(t.numpy(), d[f"{tag}_post_{k}"], rtol=1e-8, atol=1e-12)
    K = int(d["lod_count"])
    for name, key in (("emb", "embeddings"), ("log_scales", "log_scales"),
                      ("offsets", "offsets")):
        ref = np.concatenate([d[f"{tag}_post_lv{k}_{key}"] for k in range(K)])
        np.testing.assert_allclose(getattr(st, name).numpy(), ref, rtol=1e-8, atol=1e-12)


def test_adam_closed_forms():
    """Step-1/2 closed forms of the reference optimizer (test_trainer.py:139-164)."""
    p = torch.zeros(5, dtype=F64)
    m, v = torch.zeros_like(p), torch.zeros_like(p)
    oracle.adam_update(p, torch.full_like(p, 0.5), m, v, 0, 1e-2)
    np.testing.assert_allclose(p.numpy(), -1e-2 * 0.5 / (0.5 + 1e-15), rtol=1e-12)
    before = p.clone()
    oracle.adam_update(p, torch.full_like(p, -0.25), m, v, 1, 1e-2)
    mm = 0.9 * 0.05 + 0.1 * -0.25
    vv = 0.999 * 0.00025 + 0.001 * 0.0625
    step = -1e-2 * (mm / (1 - 0.81)) / (np.sqrt(vv / (1 - 0.999 ** 2)) + 1e-15)
    np.testing.assert_allclose((p - before).numpy(), step, rtol=1e-12)


@pytest.mark.slow
def test_oracle_cfg1_matches_reference(cfg1_golden):
    """Survey cfg1 (10,198 anchors x 10, 128^2): masks, order, lists, image, grads."""
    d = cfg1_golden
    from paper_2503_23044_b200.synthetic import cfg1_scene
    scene, views, images = cfg1_scene()
    np.testing.assert_array_equal(scene.levels[0].grid, d["grid0"])
    assert scene.lod_ref_distance == float(d["lod_ref"])
    centers = scene.flat_centers()
    levels = scene.flat_levels()
    cams = [oracle.Cam.of(v) for v in views]
    for i, cam in enumerate(cams):
        np.testing.assert_array_equal(
            oracle.cull(centers, levels, 1, scene.lod_ref_distance, 0, cam), d[f"mask{i}"])
    st = oracle.OracleState.create(
        centers, levels, 1, scene.lod_ref_distance, 0, 0.02, 10,
        oracle.decoder_init(10, 0, float(np.log(0.125 * 0.02))), scene.flat("embeddings"),
        np.log(scene.flat("scales")), scene.flat("offsets"), total_steps=100)
    img = oracle.render_view(st, cams[0])
    np.testing.assert_array_equal(img["splats"]["gid"], d["v0_spl_gid"])
    np.testing.assert_array_equal(img["lists"], d["v0_tile_list"])
    np.testing.assert_allclose(img["rgb"].numpy(), d["v0_img_rgb"], atol=1e-10)
    rep = oracle.train_step(st, cams, images)
    assert rep["rgb"] == pytest.approx(float(d["report_rgb"][0]), rel=1e-10)
    assert rep["rgb"] == pytest.approx(float(d["loss0"]), rel=1e-10)
    for k, t in st.weights.items():
        _grad_close(st.last_grads[f"dec/{k}"].numpy(), d[f"grad_{k}"], rel=1e-7, floor=1e-14)
    rows = d["rows"]
    for name in ("emb", "log_scales", "offsets"):
        _grad_close(st.last_grads[name].numpy()[rows], d[f"lgrad_{name}"], rel=1e-7, floor=1e-14)
    rep = oracle.train_step(st, cams, images)
    assert rep["rgb"] == pytest.approx(float(d["report_rgb"][1]), rel=1e-9)
    for k, t in st.weights.items():   # step-2 gradients (at the post-step-1 parameters)
        _grad_close(st.last_grads[f"dec/{k}"].numpy(), d[f"grad2_{k}"], rel=1e-7, floor=1e-14)
    for name in ("emb", "log_scales", "offsets"):
        _grad_close(st.last_grads[name].numpy()[rows], d[f"lgrad2_{name}"], rel=1e-7,
                    floor=1e-14)
    for k, t in st.weights.items():
        np.testing.assert_allclose(t.numpy(), d[f"post_{k}"], rtol=1e-7, atol=1e-12)
    for name in ("emb", "log_scales", "offsets"):
        np.testing.assert_allclose(getattr(st, name).numpy()[rows], d[f"post_lv_{name}"],
                                   rtol=1e-7, atol=1e-12)


@pytest.mark.slow
def test_oracle_empty_and_ragged_views_match_reference():
    """A ragged 37x29 view (partial tiles on both axes) next to a regular one:
    oracle losses and decoder update vs the reference (edge_views golden)."""
    from conftest import golden_scene, golden_view
    from paper_2503_23044_b200.geometry import CameraView, look_at
    d = load_golden("train_small")
    g = load_golden("edge_views")
    scene = golden_scene(d)
    v0 = golden_view(d, "v0", 0)
    r, t = look_at(np.array([0.0, 0.0, 5.0]), np.array([0.0, 0.0, 10.0]))
    away = CameraView(7, 48, 40, 40.0, 40.0, 23.5, 19.5, r, t)
    rr, tt = look_at(np.array([1.2, -1.1, 1.3]), np.zeros(3))
    ragged = CameraView(8, 37, 29, 30.0, 30.0, 18.0, 14.0, rr, tt)
    del away  # the reference itself raises on an empty view (see make_edge_views)
    cams = [oracle.Cam.of(v) for v in (v0, ragged)]
    images = [d["img0"], g["img_ragged"]]
    w = oracle.decoder_init(3, 0, float(np.log(0.125 * scene.base_voxel_size)))
    st = oracle.OracleState.create(
        scene.flat_centers(), scene.flat_levels(), scene.lod_count, scene.lod_ref_distance,
        scene.lod_bias, scene.base_voxel_size, 3, w, scene.flat("embeddings"),
        np.log(scene.flat("scales")), scene.flat("offsets"), total_steps=8)
    for s in range(2):
        rep = oracle.train_step(st, cams, images)
        np.testing.assert_allclose([rep["total"], rep["rgb"], rep["gaussians"]], g["loss"][s],
                                   rtol=1e-10)
    for name, t_ in st.weights.items():
        np.testing.assert_allclose(t_.detach().numpy(), g[f"post_{name}"], rtol=1e-8,
                                   atol=1e-12)


def test_oracle_normal_prior_term_is_reference_eq9_per_channel():
    """The normal-prior L1 (no reference function) is pinned on the reference's
    own Eq. 9 machinery: loss_e_depth (losses.py:65-95) per normal channel,
    averaged (golden normal_prior, make_golden.make_normal_prior)."""
    g = load_golden("normal_prior")
    leaves = [torch.tensor(g[f"n{i}"], requires_grad=True) for i in range(3)]
    val, sup = oracle.normal_l1_loss(leaves, [torch.as_tensor(g[f"rv{i}"]) for i in range(3)],
                                     [g[f"p{i}"] for i in range(3)],
                                     [g[f"pv{i}"] for i in range(3)])
    assert sup == int(g["supervised"])
    assert float(val) == pytest.approx(float(g["value"]), rel=1e-12)
    grads = torch.autograd.grad(val, leaves, allow_unused=True)
    for i in range(3):
        got = np.zeros_like(g["grad"][i]) if grads[i] is None else grads[i].numpy()
        np.testing.assert_allclose(got, g["grad"][i], rtol=1e-12, atol=1e-18)


def test_oracle_train_step_normal_term_equals_full_view_autograd(train_small):
    """oracle.train_step's tile-wise normal term (value and gradients) equals
    normal_l1_loss on the whole-view render, differentiated in one autograd
    call (the reference's train_step structure, trainer.py:270-339)."""
    d = train_small
    cams = [oracle.Cam.of(golden_view(d, f"v{i}", i)) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    rng = np.random.default_rng(4)
    npri = []
    for i in range(3):
        p = rng.normal(size=(40, 48, 3))
        npri.append((p / np.linalg.norm(p, axis=-1, keepdims=True),
                     rng.uniform(size=(40, 48)) > (0.3 if i != 1 else 1.1)))
    wn = 0.5
    st = _train_state(d, total_steps=8, step2_start=8, step3_start=8)
    # one autograd call over the whole-view renders
    for p in st.params().values():
        p.requires_grad_(True)
    rgbs, nrms, vals = [], [], []
    for cam in cams:
        P, _, _ = oracle.pipeline._view_splats(st, cam, grad=True)
        off, lst = oracle.bin_tiles(P["mean2d"].detach().numpy(), P["radius"], cam.width,
                                    cam.height)
        img = oracle.raster(P, off, lst, cam)
        rgbs.append(img["rgb"]), nrms.append(img["normal"]), vals.append(img["valid"])
    nl, _ = oracle.normal_l1_loss(nrms, vals, [p for p, _ in npri], [v for _, v in npri])
    total = oracle.l1_loss(rgbs, images) + wn * nl
    names = list(st.params())
    ref = torch.autograd.grad(total, [st.params()[k] for k in names], allow_unused=True)
    for p in st.params().values():
        p.requires_grad_(False)
    rep = oracle.train_step(st, cams, images, normal_priors=npri, normal_weight=wn)
    assert rep["normal"] == pytest.approx(float(nl), rel=1e-10)
    assert rep["total"] == pytest.approx(float(total), rel=1e-10)
    for k, r in zip(names, ref):
        r = np.zeros(st.last_grads[k].shape) if r is None else r.numpy()
        _grad_close(st.last_grads[k].numpy(), r, rel=1e-8, floor=1e-15)
