"""The drop-in boundary's remaining reference API surface on the device:
decode_inputs / decode_arrays (decoder.py:142-180), rasterize_patch on
rectangles that are not tile aligned and on explicit index subsets
(renderer.py:304-344), and the StepReport fields of the simulated
multi-worker schedule (transfer_bytes / imbalance, trainer.py:264-289,
352-364) — against outputs of the unmodified reference (golden boundary)."""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import pytest
import torch

import oracle
from conftest import golden_scene, golden_view, load_golden
from gpu_util import f32r, records_from, rel_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2503_23044_b200 import _lib
    _lib.load()


def _voxels(d, count=40):
    scene = golden_scene(d)
    rng = np.random.default_rng(2)
    idx = np.sort(rng.choice(scene.total_voxels, count, replace=False))
    return (scene, scene.flat_centers()[idx], f32r(scene.flat("embeddings")[idx]),
            f32r(scene.flat("scales")[idx]), f32r(scene.flat("offsets")[idx]))


def test_decode_inputs_matches_reference_formula(scene_small):
    from paper_2503_23044_b200.decoder import decode_inputs
    scene, c, emb, _, _ = _voxels(scene_small)
    view = golden_view(scene_small, "near")
    got = decode_inputs(c, torch.as_tensor(emb).double(), view.center,
                        scene.lod_ref_distance).cpu().numpy()
    rel = c - np.asarray(view.center)
    dist = np.maximum(np.linalg.norm(rel, axis=-1, keepdims=True), 1e-12)
    want = np.concatenate([emb, dist / scene.lod_ref_distance, rel / dist], -1)
    np.testing.assert_allclose(got, want, rtol=1e-14, atol=1e-15)


def test_decode_arrays_forward_and_gradients_vs_oracle(scene_small):
    from paper_2503_23044_b200.decoder import DecoderParams, decode_arrays
    d = scene_small
    scene, c, emb, scl, off = _voxels(d)
    view = golden_view(d, "near")
    weights = {k[2:]: d[k] for k in d if k.startswith("w_")}
    params = DecoderParams.from_arrays(2, weights)
    leaves = {"embeddings": torch.tensor(emb, dtype=torch.float32, device="cuda",
                                         requires_grad=True),
              "scales": torch.tensor(scl, dtype=torch.float32, device="cuda",
                                     requires_grad=True),
              "offsets": torch.tensor(off, dtype=torch.float32, device="cuda",
                                      requires_grad=True)}
    out = decode_arrays(params, c, leaves["embeddings"], leaves["scales"], leaves["offsets"],
                        view, scene.lod_ref_distance, 3 * scene.base_voxel_size)
    w64 = {k: torch.tensor(f32r(v)) for k, v in weights.items()}
    lv64 = {k: torch.tensor(v.detach().double().cpu().numpy(), requires_grad=True)
            for k, v in leaves.items()}
    ref = oracle.decode(w64, c, lv64["embeddings"], lv64["scales"], lv64["offsets"],
                        view.center, scene.lod_ref_distance, 3 * scene.base_voxel_size, 2)
    for k in ("means", "opacities", "colors", "scales", "quats", "normals"):
        assert tuple(out[k].shape) == tuple(ref[k].shape), k
        np.testing.assert_allclose(out[k].detach().double().cpu().numpy(),
                                   ref[k].detach().numpy(), rtol=2e-5, atol=2e-6, err_msg=k)
    rng = np.random.default_rng(4)
    cot = {k: rng.normal(size=tuple(ref[k].shape)) for k in ("means", "opacities", "colors")}
    obj = sum((out[k].double() * torch.as_tensor(v, device="cuda")).sum() for k, v in cot.items())
    got = torch.autograd.grad(obj, list(leaves.values()))
    obj64 = sum((ref[k] * torch.as_tensor(v)).sum() for k, v in cot.items())
    want = torch.autograd.grad(obj64, list(lv64.values()))
    for name, g, w in zip(leaves, got, want):
        ok, worst, nbad = rel_close(g.double().cpu().numpy(), w.numpy(), 1e-3,
                                    1e-6 * float(w.abs().max()))
        assert ok, f"{name}: {nbad} bad, worst rel {worst:.3g}"


def _golden_splats(d, tag):
    from paper_2503_23044_b200.renderer import ProjectedSplats
    spl = {k: d[f"{tag}_spl_{k}"] for k in ("mean2d", "conic", "color", "opacity",
                                             "normal_cam", "plane_d", "radius", "zkey")}
    P = records_from(spl)
    batch = SimpleNamespace(gid=d[f"{tag}_spl_gid"], owner=np.zeros(P.count, np.int32),
                            leaves=None)
    return ProjectedSplats(P, batch, None, golden_view(d, tag, 1))


def test_rasterize_patch_matches_reference_on_unaligned_rects(scene_small):
    from paper_2503_23044_b200.partition import PatchRect
    from paper_2503_23044_b200.renderer import rasterize_patch, splats_for_rect
    g = load_golden("boundary")
    splats = _golden_splats(scene_small, "near")
    view = splats.view
    for i in range(4):
        x0, y0, w, h = (int(v) for v in g[f"rect{i}"])
        np.testing.assert_array_equal(splats_for_rect(splats, x0, y0, w, h), g[f"rect{i}_idx"])
        out = rasterize_patch(PatchRect(view.view_id, i, x0, y0, w, h), splats, view)
        valid = g[f"rect{i}_valid"]
        np.testing.assert_array_equal(out["valid"].cpu().numpy(), valid)
        for k in ("rgb", "alpha", "normal"):
            err = np.abs(out[k].cpu().numpy() - g[f"rect{i}_{k}"]).max()
            assert err <= 1e-4, (i, k, err)
        derr = np.abs(out["depth"].cpu().numpy() - g[f"rect{i}_depth"])[valid].max()
        assert derr <= 1e-4, (i, derr)
    out = rasterize_patch(PatchRect(view.view_id, 9, 5, 3, 21, 13), splats, view,
                          indices=g["sub_idx"])
    for k in ("rgb", "alpha"):
        assert np.abs(out[k].cpu().numpy() - g[f"sub_{k}"]).max() <= 1e-4, k


def test_rasterize_patch_of_a_tile_equals_the_view(scene_small):
    """A tile-aligned 16x16 patch with the tile's bin list is that tile of
    rasterize_view (the reference's stitching property, test_renderer.py:229-243)."""
    from paper_2503_23044_b200.partition import PatchRect
    from paper_2503_23044_b200.renderer import bin_splats, rasterize_patch, rasterize_view
    splats = _golden_splats(scene_small, "near")
    view = splats.view
    full, _ = rasterize_view(splats, view)
    lists = bin_splats(splats, view.width, view.height)
    txn = (view.width + 15) // 16
    for t in (0, 3, 5):
        ty, tx = divmod(t, txn)
        w, h = min(16, view.width - 16 * tx), min(16, view.height - 16 * ty)
        out = rasterize_patch(PatchRect(view.view_id, t, 16 * tx, 16 * ty, w, h), splats, view,
                              indices=lists[t])
        sl = (slice(16 * ty, 16 * ty + h), slice(16 * tx, 16 * tx + w))
        for k in ("rgb", "alpha", "depth", "normal"):
            np.testing.assert_allclose(out[k].cpu().numpy(), getattr(full, k)[sl].cpu().numpy(),
                                       rtol=0, atol=1e-6, err_msg=k)


@pytest.mark.parametrize("workers", [2, 3])
def test_step_report_transfer_bytes_match_reference(train_small, workers):
    from paper_2503_23044_b200.trainer import TrainConfig, TrainState, train_step
    g = load_golden("boundary")
    d = train_small
    views = [golden_view(d, f"v{i}", i) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    st = TrainState(golden_scene(d), TrainConfig(total_steps=8, batch_size=3, workers=workers,
                                                 step2_start=8, step3_start=8, growth_stop=0))
    for s in range(2):
        rep = train_step(st, views, images)
        # step 0 schedules from the cold cost model (pixel counts, the same on
        # both sides); later steps follow each side's own measured timings
        if s == 0:
            assert rep.transfer_bytes == int(g[f"w{workers}_transfer"][s])
        else:
            assert 0 < rep.transfer_bytes <= rep.gaussians * 136 * workers
        assert rep.rgb == pytest.approx(float(g[f"w{workers}_rgb"][s]), rel=2e-4)
        assert np.isfinite(rep.imbalance) and 1.0 <= rep.imbalance <= workers


def test_tile_row_bands_compose_the_view():
    """vsx_loss_desc.tile_row0 / tile_rows (the sharded step's bands when a
    batch has fewer views than ranks): every band's pixels equal the
    full-view render bit for bit, the bands' loss sums / counts add up to the
    view's, and the bands' per-splat gradients (each normalised by the
    view's counts) sum to the full view's."""
    import bench
    from paper_2503_23044_b200 import device as D
    from paper_2503_23044_b200._lib import VsxLossDesc
    from paper_2503_23044_b200.dist import CudaShardBackend
    from paper_2503_23044_b200.trainer import TrainConfig, TrainState
    scene, views, _desc, _ = bench.workload("cfg1")
    v = views[0]
    st = TrainState(scene, TrainConfig(total_steps=100, step2_start=0, step3_start=100,
                                       growth_stop=0))
    ds = st.dscene
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    act = ds.active(v)
    dec = D.decode(st.params.abi(), st.n, act, ds.centers, st.anchors.emb, st.anchors.log_scales,
                   st.anchors.offsets, v, ds.lod_ref, ds.max_scale, status, keep_cache=False)
    P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, v, status)
    B = D.bin_tiles(P, v.width, v.height)
    H, W = v.height, v.width
    g = torch.Generator(device="cuda").manual_seed(1)
    gt = torch.rand((H, W, 3), device="cuda", generator=g)

    def run(band, counts=None):
        sums = torch.zeros(3, dtype=torch.float64, device="cuda")
        cnt = torch.zeros(2, dtype=torch.int32, device="cuda")
        loss = VsxLossDesc(gt_rgb=gt.data_ptr(), rgb_scale=1.0 / (H * W * 3),
                           sums=sums.data_ptr(), counts=cnt.data_ptr(),
                           tile_row0=band[0], tile_rows=band[1])
        R = D.raster_forward(P, B, v, loss=loss)
        if counts is not None:
            cnt.copy_(counts)
        gs = D.raster_backward(P, B, v, R, loss=loss)
        torch.cuda.synchronize()
        return R, sums, cnt, gs

    R0, s0, c0, g0 = run((0, 0))
    bands = CudaShardBackend.band_rows(v, 3)
    assert len(bands) == 3 and sum(r for _, r in bands) == (H + 15) // 16
    tot = torch.zeros(3, dtype=torch.float64, device="cuda")
    gsum = torch.zeros_like(g0)
    for r0, nr in bands:
        Rb, sb, cb, gb = run((r0, nr), counts=c0)
        y0, y1 = 16 * r0, min(H, 16 * (r0 + nr))
        assert torch.equal(Rb.rgb[y0:y1], R0.rgb[y0:y1])
        assert torch.equal(Rb.t_final[y0:y1], R0.t_final[y0:y1])
        tot += sb
        gsum += gb
    assert torch.allclose(tot, s0, rtol=1e-12, atol=0)
    rms = g0.double().pow(2).mean().sqrt()
    assert float((gsum.double() - g0.double()).abs().max()) <= 1e-5 * float(rms) + 1e-4 * \
        float(g0.double().abs().max())
