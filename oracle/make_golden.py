"""Generate tests/golden/*.npz from the UNMODIFIED reference implementation.

Run in the build container only (it imports ``/root/reference/pkg/src``,
which does not exist on the GPU box):

    python oracle/make_golden.py            # writes tests/golden/*.npz

The fixtures pin ``oracle/pipeline.py`` (see tests/test_oracle_golden.py).
Every array here is produced by calling the reference's own public functions;
nothing is recomputed by this repository's code.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np
import torch

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import voxsplat  # noqa: F401
    from voxsplat import decoder, geometry, partition, renderer, scene, trainer, losses
    return decoder, geometry, partition, renderer, scene, trainer, losses


def _view_arrays(prefix: str, view) -> dict:
    return {f"{prefix}_r": view.r, f"{prefix}_t": view.t,
            f"{prefix}_intr": np.array([view.fx, view.fy, view.cx, view.cy]),
            f"{prefix}_size": np.array([view.width, view.height]),
            f"{prefix}_center": view.center}


def _csr(tiles) -> tuple[np.ndarray, np.ndarray]:
    counts = np.array([len(t) for t in tiles], np.int64)
    offsets = np.concatenate([[0], np.cumsum(counts)])
    lists = np.concatenate([np.asarray(t, np.int64) for t in tiles]) if len(tiles) else np.zeros(0)
    return offsets, lists.astype(np.int64)


def _scene_arrays(scene) -> dict:
    out = {"lod_ref": np.array(scene.lod_ref_distance), "lod_bias": np.array(scene.lod_bias),
           "base_voxel": np.array(scene.base_voxel_size), "n": np.array(scene.offsets_per_voxel),
           "lod_count": np.array(scene.lod_count)}
    for k, lv in enumerate(scene.levels):
        out[f"grid{k}"] = lv.grid
        out[f"emb{k}"] = lv.embeddings
        out[f"off{k}"] = lv.offsets
        out[f"scl{k}"] = lv.scales
    return out


def _render_dump(prefix, renderer, view, scene, asg, params) -> dict:
    out = {}
    from voxsplat.decoder import decode_active
    batch = decode_active(params, scene, view)
    out.update({f"{prefix}_dec_{k}": getattr(batch, k).numpy()
                for k in ("means", "opacities", "colors", "scales", "quats", "normals")})
    out[f"{prefix}_dec_gid"] = batch.gid
    splats = renderer.project_splats(batch, view)
    out.update({f"{prefix}_spl_{k}": getattr(splats, k).numpy()
                for k in ("mean2d", "conic", "color", "opacity", "normal_cam", "plane_d")})
    out.update({f"{prefix}_spl_{k}": getattr(splats, k) for k in ("radius", "zkey", "gid")})
    off, lists = _csr(renderer.bin_splats(splats, view.width, view.height))
    out[f"{prefix}_tile_off"], out[f"{prefix}_tile_list"] = off, lists
    targets, counts = renderer.rasterize_view(splats, view)
    for k in ("rgb", "depth", "normal", "alpha", "valid", "raw_normal"):
        out[f"{prefix}_img_{k}"] = getattr(targets, k).numpy()
    out[f"{prefix}_counts"] = counts
    return out


def make_scene_small():
    decoder, geometry, partition, renderer, scene_m, trainer, _ = _ref()
    rng = np.random.default_rng(0)
    pts = scene_m.SparsePoints(positions=rng.uniform(-1, 1, size=(150, 3)))
    scene = scene_m.build_hierarchy(pts, 0.5, 3, offsets_per_voxel=2, seed=0)
    r, t = geometry.look_at(np.array([0.0, -3.0, 1.0]), np.zeros(3))
    far = geometry.CameraView(0, 48, 48, 40.0, 40.0, 23.5, 23.5, r, t)
    r2, t2 = geometry.look_at(np.array([0.3, -1.2, 0.6]), np.array([0.0, 0.2, 0.0]))
    near = geometry.CameraView(1, 40, 36, 30.0, 30.0, 19.5, 17.5, r2, t2)
    scene.set_lod_reference([far])
    params = decoder.DecoderParams.init(2, seed=0, scale_bias=float(np.log(0.1)))
    asg = partition.assign_voxels(scene, 1)
    out = {"points": pts.positions, **_scene_arrays(scene), **_view_arrays("far", far),
           **_view_arrays("near", near)}
    for name, t_ in params.tensors.items():
        out[f"w_{name}"] = t_.numpy()
    for tag, view in (("far", far), ("near", near)):
        for k in range(scene.lod_count):
            out[f"{tag}_mask{k}"] = scene_m.active_mask(scene, k, view)
        out.update(_render_dump(tag, renderer, view, scene, asg, params))
    np.savez_compressed(OUT / "scene_small.npz", **out)


def _leaf_case(rng, count, view):
    """Random gaussians in front of an identity camera with mixed sizes."""
    z = rng.uniform(1.2, 4.0, size=count)
    u = rng.uniform(-4.0, view.width + 4.0, size=count)
    v = rng.uniform(-4.0, view.height + 4.0, size=count)
    means = np.stack([(u - view.cx) / view.fx * z, (v - view.cy) / view.fy * z, z], -1)
    scales = rng.uniform(0.01, 0.25, size=(count, 3))
    quats = rng.normal(size=(count, 4))
    quats /= np.linalg.norm(quats, axis=-1, keepdims=True)
    return {"means": means, "opacities": rng.uniform(0.05, 0.95, size=count),
            "colors": rng.uniform(0.0, 1.0, size=(count, 3)), "scales": scales,
            "quats": quats}


def make_raster_leaf():
    decoder, geometry, partition, renderer, scene_m, trainer, _ = _ref()
    out = {}
    for case, (seed, count, w, h, f) in enumerate([(1, 60, 40, 24, 30.0),
                                                   (2, 300, 64, 48, 50.0)]):
        rng = np.random.default_rng(seed)
        view = geometry.CameraView(case, w, h, f, f, (w - 1) / 2.0, (h - 1) / 2.0,
                                   np.eye(3), np.zeros(3))
        arr = _leaf_case(rng, count, view)
        batch = renderer.make_leaf_gaussians(arr["means"], arr["opacities"], arr["colors"],
                                             arr["scales"], arr["quats"], requires_grad=True)
        splats = renderer.project_splats(batch, view)
        targets, counts = renderer.rasterize_view(splats, view)
        off, lists = _csr(renderer.bin_splats(splats, view.width, view.height))
        rn = targets.raw_normal.detach().numpy()
        rx = (np.arange(w) - view.cx) / view.fx
        ry = (np.arange(h) - view.cy) / view.fy
        denom = rn[..., 0] * rx[None, :] + rn[..., 1] * ry[:, None] + rn[..., 2]
        guard = (targets.alpha.detach().numpy() > 0.05) & (np.abs(denom) > 1e-2)
        cot = {"rgb": rng.normal(size=(h, w, 3)), "alpha": rng.normal(size=(h, w)),
               "depth": rng.normal(size=(h, w)) * guard,
               "normal": rng.normal(size=(h, w, 3)) * guard[..., None]}
        grads = renderer.rasterize_backward(
            splats, {"rgb": targets.rgb, "alpha": targets.alpha, "depth": targets.depth,
                     "normal": targets.normal}, cot)
        p = f"c{case}"
        out.update({f"{p}_{k}": a for k, a in arr.items()})
        out.update(_view_arrays(p, view))
        out.update({f"{p}_spl_{k}": getattr(splats, k).detach().numpy()
                    for k in ("mean2d", "conic", "color", "opacity", "normal_cam", "plane_d")})
        out.update({f"{p}_spl_{k}": getattr(splats, k) for k in ("radius", "zkey", "gid")})
        out[f"{p}_tile_off"], out[f"{p}_tile_list"] = off, lists
        for k in ("rgb", "depth", "normal", "alpha", "valid", "raw_normal"):
            out[f"{p}_img_{k}"] = getattr(targets, k).detach().numpy()
        out.update({f"{p}_cot_{k}": c for k, c in cot.items()})
        out.update({f"{p}_grad_{k}": g.numpy() for k, g in grads.items()})
    np.savez_compressed(OUT / "raster_leaf.npz", **out)


def _cfg1_scene(scene_m, geometry):
    rng = np.random.default_rng(0)
    pts = np.stack([rng.uniform(-1, 1, 120000), rng.uniform(-1, 1, 120000),
                    rng.uniform(-0.005, 0.005, 120000)], -1)
    scene = scene_m.build_hierarchy(scene_m.SparsePoints(pts), base_voxel_size=0.02,
                                    lod_count=1, offsets_per_voxel=10, seed=0)
    f = 64.0 / np.tan(np.radians(30.0))
    views = []
    for i in range(4):
        eye = np.array([0.3 * np.cos(np.pi * i / 2), 0.3 * np.sin(np.pi * i / 2), 2.2])
        r, t = geometry.look_at(eye, np.zeros(3), up=(0.0, 1.0, 0.0))
        views.append(geometry.CameraView(i, 128, 128, f, f, 63.5, 63.5, r, t))
    scene.set_lod_reference(views)
    images = [rng.uniform(0, 1, (128, 128, 3)) for _ in range(4)]
    return scene, views, images


def _reference_grads(trainer, renderer, losses, state, views, images):
    """The reference train_step's gradient block (trainer.py:270-339), via its own API."""
    dstate = state.decode_state()
    targets, means = [], []
    for view in views:
        batch, _ = renderer.transfer_gaussians(view, state.scene, state.assignment,
                                               state.replicas[0], state=dstate,
                                               keep_graph=True)
        splats = renderer.project_splats(batch, view)
        t, _ = renderer.rasterize_view(splats, view, renderer.ALL_TASKS)
        targets.append(t)
        means.append(batch.means)
    loss = losses.bl_rgb_loss([t.rgb for t in targets],
                              [torch.as_tensor(im) for im in images])
    dec = state.replicas[0].tensors
    names = list(dec)
    lv = [state.level_state[0][k] for k in ("embeddings", "log_scales", "offsets")]
    g = torch.autograd.grad(loss, [dec[n] for n in names] + lv, allow_unused=True)
    return float(loss), {n: x.numpy() for n, x in zip(names, g[:len(names)])}, \
        [x.numpy() for x in g[len(names):]]


def make_cfg1():
    decoder, geometry, partition, renderer, scene_m, trainer, losses = _ref()
    t0 = time.time()
    torch.set_num_threads(8)
    scene, views, images = _cfg1_scene(scene_m, geometry)
    out = {"lod_ref": np.array(scene.lod_ref_distance), "grid0": scene.levels[0].grid}
    for i, v in enumerate(views):
        out[f"mask{i}"] = scene_m.active_mask(scene, 0, v)
    cfg = trainer.TrainConfig(total_steps=100, batch_size=4, workers=1, step2_start=100,
                              step3_start=100, growth_stop=0, log_every=0)
    state = trainer.make_state(scene, cfg)
    asg = state.assignment
    params = state.replicas[0]
    dump = _render_dump("v0", renderer, views[0], scene, asg, params)
    keep = ("v0_spl_zkey", "v0_spl_gid", "v0_spl_radius", "v0_tile_off", "v0_tile_list",
            "v0_img_rgb", "v0_img_depth", "v0_img_alpha", "v0_img_valid", "v0_counts")
    out.update({k: dump[k] for k in keep})
    loss, dgrads, lgrads = _reference_grads(trainer, renderer, losses, state, views, images)
    rows = np.random.default_rng(7).choice(scene.levels[0].count, 512, replace=False)
    out["loss0"] = np.array(loss)
    out.update({f"grad_{k}": a for k, a in dgrads.items()})
    out["rows"] = rows
    for name, a in zip(("emb", "log_scales", "offsets"), lgrads):
        out[f"lgrad_{name}"] = a[rows]
    reports = [trainer.train_step(state, views, images)]
    # step-2 gradients (at the post-step-1 parameters): the post-step tests
    # exclude elements whose gradient in either step is at the noise floor
    _, dgrads2, lgrads2 = _reference_grads(trainer, renderer, losses, state, views, images)
    out.update({f"grad2_{k}": a for k, a in dgrads2.items()})
    for name, a in zip(("emb", "log_scales", "offsets"), lgrads2):
        out[f"lgrad2_{name}"] = a[rows]
    reports.append(trainer.train_step(state, views, images))
    out["report_rgb"] = np.array([r.rgb for r in reports])
    for k, t_ in state.replicas[0].tensors.items():
        out[f"post_{k}"] = t_.detach().numpy()
    for name, key in (("emb", "embeddings"), ("log_scales", "log_scales"),
                      ("offsets", "offsets")):
        out[f"post_lv_{name}"] = state.level_state[0][key].detach().numpy()[rows]
    # The same two steps from float32-representable initial parameters: the
    # device's exact inputs, so its gradients are compared without the
    # input-rounding term (f32_*). The full post-step-1 parameters let the
    # device compute its step-2 gradient at the reference's parameters.
    state = trainer.make_state(scene, cfg)
    prng = np.random.default_rng(17)
    for s in range(2):
        # every step starts from float32-representable parameters, as the
        # device's do (a float64 post-step value rounded by the device could
        # flip a near-tie decision and make the step-2 gradients incomparable)
        with torch.no_grad():
            for t_ in state.replicas[0].tensors.values():
                t_.copy_(t_.float().double())
            for key in ("embeddings", "log_scales", "offsets"):
                lv = state.level_state[0][key]
                lv.copy_(lv.float().double())
        _, dg, lg = _reference_grads(trainer, renderer, losses, state, views, images)
        pre = "f32_grad" if s == 0 else "f32_grad2"
        out.update({f"{pre}_{k}": a for k, a in dg.items()})
        for name, a in zip(("emb", "log_scales", "offsets"), lg):
            out[f"f32_l{pre[4:]}_{name}"] = a[rows]
        # noise floor: the same gradient with every parameter moved by one
        # float32 ulp (random sign) -- the sensitivity of each gradient element
        # to the rounding of its inputs, which no float32 pipeline can avoid
        params = list(state.replicas[0].tensors.values()) + \
            [state.level_state[0][k] for k in ("embeddings", "log_scales", "offsets")]
        saved = [p_.detach().clone() for p_ in params]
        with torch.no_grad():
            for p_ in params:
                sgn = torch.as_tensor(prng.choice([-1.0, 1.0], size=tuple(p_.shape)))
                p_.copy_(p_ * (1.0 + sgn * 2.0 ** -23))
        _, dgp, lgp = _reference_grads(trainer, renderer, losses, state, views, images)
        with torch.no_grad():
            for p_, v_ in zip(params, saved):
                p_.copy_(v_)
        out.update({f"f32p_{pre[4:]}_{k}": a for k, a in dgp.items()})
        for name, a in zip(("emb", "log_scales", "offsets"), lgp):
            out[f"f32p_l{pre[4:]}_{name}"] = a[rows]
        rep = trainer.train_step(state, views, images)
        out[f"f32_report_rgb{s}"] = np.array(rep.rgb)
        tag = "f32_post1" if s == 0 else "f32_post"
        # copies: the next step updates the parameter tensors in place
        for k, t_ in state.replicas[0].tensors.items():
            out[f"{tag}_{k}"] = t_.detach().numpy().copy()
        for name, key in (("emb", "embeddings"), ("log_scales", "log_scales"),
                          ("offsets", "offsets")):
            a = state.level_state[0][key].detach().numpy()
            out[f"{tag}_lv_{name}"] = a.copy() if s == 0 else a[rows]
    np.savez_compressed(OUT / "cfg1.npz", **out)
    print(f"cfg1 golden in {time.time() - t0:.0f}s")


def make_train_small():
    decoder, geometry, partition, renderer, scene_m, trainer, losses = _ref()
    from voxsplat.depth_prior import EnhancedDepthMap
    rng = np.random.default_rng(3)
    pts = scene_m.SparsePoints(positions=np.concatenate([
        np.stack([rng.uniform(-1, 1, 400), rng.uniform(-1, 1, 400),
                  rng.uniform(-0.05, 0.05, 400)], -1),
        rng.uniform(-0.3, 0.3, size=(100, 3)) + np.array([0.0, 0.0, 0.3])]))
    views = []
    for i in range(3):
        ang = 2 * np.pi * i / 3
        r, t = geometry.look_at(np.array([1.6 * np.cos(ang), 1.6 * np.sin(ang), 1.4]),
                                np.zeros(3))
        views.append(geometry.CameraView(i, 48, 40, 40.0, 40.0, 23.5, 19.5, r, t))
    scene = scene_m.build_hierarchy(pts, 0.25, 2, offsets_per_voxel=3, seed=4, views=views)
    out = {"points": pts.positions, **_scene_arrays(scene)}
    for i, v in enumerate(views):
        out.update(_view_arrays(f"v{i}", v))
    images = [rng.uniform(0, 1, (40, 48, 3)) for _ in views]
    priors = []
    for i, v in enumerate(views):
        d = rng.uniform(1.0, 2.5, (40, 48))
        valid = rng.uniform(size=(40, 48)) > 0.25
        priors.append(EnhancedDepthMap(values=np.where(valid, d, 0.0), valid=valid,
                                       min_roundtrip=np.zeros((40, 48)), tau=1.0))
        out[f"img{i}"] = images[i]
        out[f"prior{i}"] = priors[i].values
        out[f"pvalid{i}"] = valid
    # "geo": the Eq. 10 NCC term ramps in from step 0 (w3 = 0.025, 0.05 at
    # steps 1, 2); the three views give one (reference, source) pair
    for tag, s2, s3 in (("rgb", 8, 8), ("depth", 0, 8), ("geo", 8, 0)):
        scene_t = scene_m.build_hierarchy(pts, 0.25, 2, offsets_per_voxel=3, seed=4,
                                          views=views)
        cfg = trainer.TrainConfig(total_steps=8, batch_size=3, workers=1, step2_start=s2,
                                  step3_start=s3, growth_stop=0, log_every=0)
        state = trainer.make_state(scene_t, cfg)
        reps = []
        for _ in range(3):
            reps.append(trainer.train_step(state, views, images,
                                           priors if tag == "depth" else None))
        out[f"{tag}_loss"] = np.array([[r.total, r.rgb, r.depth] for r in reps])
        out[f"{tag}_supervised"] = np.array([r.supervised_depth_px for r in reps])
        out[f"{tag}_geo"] = np.array([[r.geo, r.w3, r.geo_pairs, r.geo_patches] for r in reps])
        for k, t_ in state.replicas[0].tensors.items():
            out[f"{tag}_post_{k}"] = t_.detach().numpy()
        for k in range(scene_t.lod_count):
            for key in ("embeddings", "log_scales", "offsets"):
                out[f"{tag}_post_lv{k}_{key}"] = state.level_state[k][key].detach().numpy()
    np.savez_compressed(OUT / "train_small.npz", **out)


def make_growth():
    """f3 anchor growth (trainer.py:341-349, 379-454): the train_small scene,
    two reference train steps (growth accumulators), grow_anchors, one more
    step on the grown scene."""
    decoder, geometry, partition, renderer, scene_m, trainer, losses = _ref()
    d = np.load(OUT / "train_small.npz")
    pts = scene_m.SparsePoints(positions=d["points"])
    views = []
    for i in range(3):
        views.append(geometry.CameraView(i, int(d[f"v{i}_size"][0]), int(d[f"v{i}_size"][1]),
                                         *[float(x) for x in d[f"v{i}_intr"]],
                                         d[f"v{i}_r"], d[f"v{i}_t"]))
    images = [d[f"img{i}"] for i in range(3)]
    scene = scene_m.build_hierarchy(pts, 0.25, 2, offsets_per_voxel=3, seed=4, views=views)
    cfg = trainer.TrainConfig(total_steps=8, batch_size=3, workers=1, step2_start=8,
                              step3_start=8, growth_stop=8, growth_threshold=7.35e-4,
                              log_every=0)
    state = trainer.make_state(scene, cfg)
    out = {}
    for _ in range(2):
        trainer.train_step(state, views, images)
    for k in range(scene.lod_count):
        out[f"grow_sum{k}"] = state.grow_sum[k].copy()
        out[f"grow_cnt{k}"] = state.grow_cnt[k].copy()
    out["grown"] = np.array(trainer.grow_anchors(state))
    out["events"] = np.array([[e["level"], e["added"], e["parents"]] for e in state.grow_events])
    for k, lv in enumerate(scene.levels):
        out[f"grid{k}"] = lv.grid
        out[f"owner{k}"] = lv.owner
    rep = trainer.train_step(state, views, images)
    out["post_loss"] = np.array([rep.total, rep.rgb])
    for k, t_ in state.replicas[0].tensors.items():
        out[f"post_{k}"] = t_.detach().numpy()
    for k in range(scene.lod_count):
        for key in ("embeddings", "log_scales", "offsets"):
            out[f"post_lv{k}_{key}"] = state.level_state[k][key].detach().numpy()
    np.savez_compressed(OUT / "growth.npz", **out)


def make_fusion():
    """f4 TSDF integration (fusion.py:102-133): a volume around the
    depth_prior ground plane, integrated with the three aligned depth maps of
    that fixture; per-call touched counts and the final tsdf / weight."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from voxsplat.fusion import TsdfVolume
    from voxsplat.geometry import CameraView
    d = np.load(OUT / "depth_prior.npz")
    vol = TsdfVolume.from_bounds([-3.0, -2.0, -0.5], [3.0, 3.0, 0.5], 0.1, 0.3)
    touched = []
    for i in range(3):
        fx, fy, cx, cy = d[f"v{i}_intr"]
        w, h = d[f"v{i}_size"]
        view = CameraView(i, int(w), int(h), float(fx), float(fy), float(cx), float(cy),
                          d[f"v{i}_r"], d[f"v{i}_t"])
        touched.append(vol.integrate(d[f"aligned{i}_values"], d[f"aligned{i}_valid"], view))
    np.savez_compressed(OUT / "fusion.npz", touched=np.array(touched), dims=np.array(vol.dims),
                        origin=vol.origin, voxel=np.array(vol.voxel_size),
                        trunc=np.array(vol.truncation), tsdf=vol.tsdf, weight=vol.weight)


def make_checkpoint():
    """f4 .vsnap state IO (snapshot.py, trainer.py:491-522): a reference
    checkpoint after two train steps on the train_small scene (the raw file,
    committed), the records its own reader returns, and the reference's loss
    and parameters after one more step from that file."""
    decoder, geometry, partition, renderer, scene_m, trainer, losses = _ref()
    from voxsplat import snapshot
    d = np.load(OUT / "train_small.npz")
    pts = scene_m.SparsePoints(positions=d["points"])
    views = [geometry.CameraView(i, int(d[f"v{i}_size"][0]), int(d[f"v{i}_size"][1]),
                                 *[float(x) for x in d[f"v{i}_intr"]], d[f"v{i}_r"],
                                 d[f"v{i}_t"]) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    scene = scene_m.build_hierarchy(pts, 0.25, 2, offsets_per_voxel=3, seed=4, views=views)
    cfg = trainer.TrainConfig(total_steps=8, batch_size=3, workers=1, step2_start=8,
                              step3_start=8, growth_stop=0, log_every=0)
    state = trainer.make_state(scene, cfg)
    for _ in range(2):
        trainer.train_step(state, views, images)
    path = OUT / "checkpoint.vsnap"
    trainer.save_checkpoint(path, state)
    data = snapshot.read_snapshot(path)
    out = {f"{tag}:{name}": arr for tag, rec in data.items() for name, arr in rec.items()}
    # resume: scene + decoder from the file, train records restored
    scene2, dec2, rest = snapshot.load_scene(path)
    st2 = trainer.make_state(scene2, cfg)
    with torch.no_grad():
        for k, t_ in st2.replicas[0].tensors.items():
            t_.copy_(dec2.tensors[k])
    trainer.restore_train_records(st2, rest["TRN1"])
    rep = trainer.train_step(st2, views, images)
    out["resume_loss"] = np.array([rep.total, rep.rgb, rep.step])
    for k, t_ in st2.replicas[0].tensors.items():
        out[f"resume_post_{k}"] = t_.detach().numpy()
    for k in range(scene2.lod_count):
        for key in ("embeddings", "log_scales", "offsets"):
            out[f"resume_post_lv{k}_{key}"] = st2.level_state[k][key].detach().numpy()
    np.savez_compressed(OUT / "checkpoint.npz", **out)


def make_partition():
    """f4 LPT/EMA scheduler (partition.py:84-207): schedules of three views
    over 3 workers, cold and after two epochs of random measured seconds."""
    decoder, geometry, partition, renderer, scene_m, trainer, losses = _ref()
    rng = np.random.default_rng(21)
    views = [geometry.CameraView(i, int(w), int(h), 50.0, 50.0, (w - 1) / 2, (h - 1) / 2,
                                 np.eye(3), np.zeros(3))
             for i, (w, h) in enumerate([(70, 40), (48, 48), (33, 65)])]
    pts = scene_m.SparsePoints(positions=rng.uniform(-1, 1, size=(300, 3)))
    scene = scene_m.build_hierarchy(pts, 0.5, 2, offsets_per_voxel=2, seed=0)
    asg = partition.assign_voxels(scene, 3)
    model = partition.PatchCostModel()
    out = {"lpt_costs": rng.uniform(0, 5, 40).round(1)}
    out["lpt_workers"] = partition.lpt_assign(out["lpt_costs"], 4)
    for ep in range(3):
        sch = partition.schedule_patches(views, 3, model)
        out[f"ep{ep}_workers"] = sch.workers
        out[f"ep{ep}_est"] = sch.est_costs
        out[f"ep{ep}_loads"] = sch.loads()
        meas = rng.uniform(0.0, 2e-3, len(sch.patches))
        out[f"ep{ep}_measured"] = meas
        st = partition.balance_report(asg, sch, meas, epoch=ep, cost_model=model)
        out[f"ep{ep}_seconds"] = st.seconds
        out[f"ep{ep}_stats"] = np.array([st.imbalance, st.load_fraction])
        out[f"ep{ep}_voxels"] = st.voxel_counts
    for k, lv in enumerate(scene.levels):
        out[f"grid{k}"] = lv.grid
    np.savez_compressed(OUT / "partition.npz", **out)


def make_edge_views():
    """Edge cases of train_step: a view that sees no anchor and a ragged
    37x29 view next to a regular one (train_small scene); the reference's
    losses of two steps."""
    decoder, geometry, partition, renderer, scene_m, trainer, losses = _ref()
    d = np.load(OUT / "train_small.npz")
    pts = scene_m.SparsePoints(positions=d["points"])
    v0 = geometry.CameraView(0, int(d["v0_size"][0]), int(d["v0_size"][1]),
                             *[float(x) for x in d["v0_intr"]], d["v0_r"], d["v0_t"])
    views0 = [geometry.CameraView(i, int(d[f"v{i}_size"][0]), int(d[f"v{i}_size"][1]),
                                  *[float(x) for x in d[f"v{i}_intr"]], d[f"v{i}_r"],
                                  d[f"v{i}_t"]) for i in range(3)]
    r, t = geometry.look_at(np.array([0.0, 0.0, 5.0]), np.array([0.0, 0.0, 10.0]))
    away = geometry.CameraView(7, 48, 40, 40.0, 40.0, 23.5, 19.5, r, t)
    rr, tt = geometry.look_at(np.array([1.2, -1.1, 1.3]), np.zeros(3))
    ragged = geometry.CameraView(8, 37, 29, 30.0, 30.0, 18.0, 14.0, rr, tt)
    rng = np.random.default_rng(5)
    images = [d["img0"], rng.uniform(0, 1, (40, 48, 3)), rng.uniform(0, 1, (29, 37, 3))]
    scene = scene_m.build_hierarchy(pts, 0.25, 2, offsets_per_voxel=3, seed=4, views=views0)
    cfg = trainer.TrainConfig(total_steps=8, batch_size=3, workers=1, step2_start=8,
                              step3_start=8, growth_stop=0, log_every=0)
    state = trainer.make_state(scene, cfg)
    # the reference raises inside autograd.grad on a view with no active
    # anchor (its decoded means do not require grad), so the golden uses the
    # regular + ragged views; the empty view is checked against the oracle
    del away
    images = [images[0], images[2]]
    reps = [trainer.train_step(state, [v0, ragged], images) for _ in range(2)]
    out = {"loss": np.array([[r_.total, r_.rgb, r_.gaussians] for r_ in reps]),
           "img_ragged": images[1]}
    for k, t_ in state.replicas[0].tensors.items():
        out[f"post_{k}"] = t_.detach().numpy()
    np.savez_compressed(OUT / "edge_views.npz", **out)


def make_depth_prior():
    """f1 prior precompute: three aerial views of the ground plane z = 0 with
    raw relative depth maps (planted affine + noise, a corrupted stripe in view
    0) and sparse plane points; outputs of the reference's fit_scale_shift,
    apply_scale_shift, select_neighbors, reprojection_error and enhance."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from voxsplat import depth_prior as dp
    from voxsplat.geometry import CameraView, look_at
    rng = np.random.default_rng(11)
    W, H, f = 64, 48, 55.0
    eyes = [(0.0, -4.0, 6.0), (1.0, -4.2, 6.1), (-1.2, -3.8, 5.9)]
    views = []
    for i, e in enumerate(eyes):
        r, t = look_at(np.array(e), np.array([0.1 * i, 0.5, 0.0]))
        views.append(CameraView(view_id=i, width=W, height=H, fx=f, fy=f, cx=(W - 1) / 2.0,
                                cy=(H - 1) / 2.0, r=r, t=t))
    uu, vv = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    raws, metrics = [], []
    st = [(0.8, 0.3), (1.25, -0.2), (0.6, 0.45)]
    for i, v in enumerate(views):
        d = np.stack([(uu - v.cx) / v.fx, (vv - v.cy) / v.fy, np.ones_like(uu)], -1)
        dw = d @ v.r                      # camera ray -> world direction (r rows = axes)
        c = v.center
        metric = -c[2] / dw[..., 2]       # camera z of the plane hit (ray has unit cam z)
        s, b = st[i]
        raw = (metric - b) / s + rng.normal(0.0, 1e-3, metric.shape)
        if i == 0:
            raw[30:34, :] *= 1.3          # corrupted stripe
        raws.append(raw)
        metrics.append(metric)
    pts = np.stack([rng.uniform(-3, 3, 400), rng.uniform(-2, 3, 400), np.zeros(400)], -1)
    out = {"raw0": raws[0], "raw1": raws[1], "raw2": raws[2], "points": pts,
           "metric0": metrics[0]}
    for i, v in enumerate(views):
        out.update(_view_arrays(f"v{i}", v))
    aligned = []
    for i, v in enumerate(views):
        fit = dp.fit_scale_shift(raws[i], v, pts)
        out[f"fit{i}"] = np.array([fit.scale, fit.shift, fit.samples, fit.inliers], np.float64)
        al = dp.apply_scale_shift(raws[i], fit)
        aligned.append(al)
        out[f"aligned{i}_values"] = al.values
        out[f"aligned{i}_valid"] = al.valid
    nb0 = dp.select_neighbors(views, 0)
    out["neighbors0"] = np.array(nb0, np.int64)
    out["err01"] = dp.reprojection_error(aligned[0], views[0], aligned[1], views[1])
    enh = dp.enhance(aligned[0], views[0], [(aligned[j], views[j]) for j in nb0], tau=1.0)
    out["enh0_values"] = enh.values
    out["enh0_valid"] = enh.valid
    out["enh0_min_roundtrip"] = enh.min_roundtrip
    np.savez_compressed(OUT / "depth_prior.npz", **out)


def make_normal_prior():
    """The normal-prior L1 of the RGB-D-N objective has no reference function
    (the reference supervises normals through the depth quotient and Eq. 10);
    its contract is Eq. 9 applied per channel: the reference's own
    loss_e_depth (losses.py:65-95) on each of the 3 normal channels, averaged.
    Three views of random unit normals, render-valid and prior-valid masks."""
    decoder, geometry, partition, renderer, scene_m, trainer, losses = _ref()
    rng = np.random.default_rng(21)
    H, W = 24, 32
    out = {}
    normals, rvalid, priors, pvalid = [], [], [], []
    for i in range(3):
        n = rng.normal(size=(H, W, 3))
        n /= np.linalg.norm(n, axis=-1, keepdims=True)
        p = rng.normal(size=(H, W, 3))
        p /= np.linalg.norm(p, axis=-1, keepdims=True)
        rv = rng.uniform(size=(H, W)) > 0.2
        pv = rng.uniform(size=(H, W)) > (0.3 if i < 2 else 1.1)   # view 2: no prior pixel
        normals.append(n), rvalid.append(rv), priors.append(p), pvalid.append(pv)
        out.update({f"n{i}": n, "rv%d" % i: rv, f"p{i}": p, f"pv{i}": pv})
    vals, grads, sup = [], np.zeros((3, H, W, 3)), 0
    for c in range(3):
        v, g, s_ = losses.loss_e_depth([n[..., c] for n in normals], rvalid,
                                       [p[..., c] for p in priors], pvalid)
        vals.append(v)
        grads[..., c] = np.stack(g)
        sup = s_
    out["value"] = np.array(np.mean(vals))
    out["grad"] = grads / 3.0
    out["supervised"] = np.array(sup)
    np.savez_compressed(OUT / "normal_prior.npz", **out)


def make_geo_loss():
    """f2 Eq. 10: the reference's own render targets of two coplanar textured
    sheets (the layout of its geo FD test, helpers.py:256-300) for two texture
    phases, bl_geo_loss values / stats with a seeded rng, and the gradients of
    the loss w.r.t. the source view's rendered rgb, normal and depth; plus
    reference picks of _stratified_centers on random candidate sets."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    tests_dir = str(Path(REF).parent / "tests")
    if tests_dir not in sys.path:
        sys.path.insert(0, tests_dir)
    import helpers as H
    from voxsplat import losses as L
    from voxsplat.geometry import CameraView
    from voxsplat.renderer import make_leaf_gaussians, project_splats, rasterize_view
    out = {}
    for case, (phase_b, tilt) in enumerate([(4.0, (0.05, -0.08)), (1.0, (-0.1, 0.07))]):
        normal = np.array([tilt[0], tilt[1], 1.0])
        point = np.array([0.0, 0.0, 2.2])
        src_view = CameraView(view_id=0, width=24, height=24, fx=30.0, fy=30.0, cx=11.5, cy=11.5,
                              r=np.eye(3), t=np.zeros(3))
        ref_view = CameraView(view_id=1, width=40, height=40, fx=30.0, fy=30.0, cx=19.5,
                              cy=19.5, r=np.eye(3), t=-np.array([0.06, 0.04, 0.0]))
        targets = []
        for view, phase in ((ref_view, phase_b), (src_view, 1.0)):
            arrays = H.plane_gaussian_arrays(normal, point, extent=2.0, spacing=0.18)
            arrays["colors"] = H._smooth_colors(arrays["means"], phase)
            batch = make_leaf_gaussians(arrays["means"], arrays["opacities"], arrays["colors"],
                                        arrays["scales"], arrays["quats"], requires_grad=True)
            t, _ = rasterize_view(project_splats(batch, view), view)
            targets.append(t)
        views = [ref_view, src_view]
        val, stats = L.bl_geo_loss(targets, views, np.random.default_rng(case), patch_count=16)
        src = targets[1]
        g = torch.autograd.grad(val, [src.rgb, src.normal, src.depth], allow_unused=True)
        p = f"c{case}_"
        for k, t in zip(("ref", "src"), targets):
            for f in ("rgb", "normal", "depth", "alpha"):
                out[p + f"{k}_{f}"] = getattr(t, f).detach().numpy()
            out[p + f"{k}_valid"] = t.valid.numpy()
        out.update(_view_arrays(p + "vref", ref_view))
        out.update(_view_arrays(p + "vsrc", src_view))
        out[p + "loss"] = np.array(float(val))
        out[p + "stats"] = np.array([stats.pairs_used, stats.patches_used,
                                     stats.patches_rejected])
        for name, gg, like in zip(("g_rgb", "g_normal", "g_depth"), g,
                                  (src.rgb, src.normal, src.depth)):
            out[p + name] = (gg if gg is not None else torch.zeros_like(like)).detach().numpy()
    rng = np.random.default_rng(5)
    for k in range(4):
        n = int(rng.integers(20, 400))
        w, h = int(rng.integers(16, 80)), int(rng.integers(16, 80))
        cu = rng.integers(0, w, n).astype(np.float64)
        cv = rng.integers(0, h, n).astype(np.float64)
        cnt = int(rng.integers(4, 70))
        out[f"strat{k}_in"] = np.concatenate([cu, cv])
        out[f"strat{k}_args"] = np.array([w, h, cnt, 100 + k])
        out[f"strat{k}_out"] = L._stratified_centers(cu, cv, w, h, cnt,
                                                     np.random.default_rng(100 + k))
    np.savez_compressed(OUT / "geo_loss.npz", **out)


def make_boundary():
    """API-surface cases of the drop-in boundary: the reference's
    rasterize_patch on rectangles that are not tile aligned (scene_small
    'near' view, its own sorted splats; renderer.py:304-344), and its
    train_step report fields of the simulated multi-worker schedule
    (transfer_bytes, trainer.py:264-289) at workers = 2 and 3 on train_small."""
    decoder, geometry, partition, renderer, scene_m, trainer, _ = _ref()
    out = {}
    rng = np.random.default_rng(0)
    pts = scene_m.SparsePoints(positions=rng.uniform(-1, 1, size=(150, 3)))
    scene = scene_m.build_hierarchy(pts, 0.5, 3, offsets_per_voxel=2, seed=0)
    r, t = geometry.look_at(np.array([0.0, -3.0, 1.0]), np.zeros(3))
    far = geometry.CameraView(0, 48, 48, 40.0, 40.0, 23.5, 23.5, r, t)
    r2, t2 = geometry.look_at(np.array([0.3, -1.2, 0.6]), np.array([0.0, 0.2, 0.0]))
    near = geometry.CameraView(1, 40, 36, 30.0, 30.0, 19.5, 17.5, r2, t2)
    scene.set_lod_reference([far])
    params = decoder.DecoderParams.init(2, seed=0, scale_bias=float(np.log(0.1)))
    from voxsplat.decoder import decode_active
    splats = renderer.project_splats(decode_active(params, scene, near), near)
    rects = [(5, 3, 21, 13), (0, 0, 40, 36), (17, 20, 9, 16), (30, 1, 10, 7)]
    for i, (x0, y0, w, h) in enumerate(rects):
        rect = partition.PatchRect(near.view_id, i, x0, y0, w, h)
        res = renderer.rasterize_patch(rect, splats, near)
        out[f"rect{i}"] = np.array([x0, y0, w, h])
        out[f"rect{i}_idx"] = renderer.splats_for_rect(splats, x0, y0, w, h)
        for k, v in res.items():
            out[f"rect{i}_{k}"] = v.detach().numpy()
    # an explicit index subset (every other overlapping splat)
    idx = renderer.splats_for_rect(splats, 5, 3, 21, 13)[::2]
    res = renderer.rasterize_patch(partition.PatchRect(near.view_id, 9, 5, 3, 21, 13), splats,
                                   near, indices=idx)
    out["sub_idx"] = idx
    for k, v in res.items():
        out[f"sub_{k}"] = v.detach().numpy()
    d = np.load(OUT / "train_small.npz")
    tpts = scene_m.SparsePoints(positions=d["points"])
    views = []
    for i in range(3):
        ang = 2 * np.pi * i / 3
        rr, tt = geometry.look_at(np.array([1.6 * np.cos(ang), 1.6 * np.sin(ang), 1.4]),
                                  np.zeros(3))
        views.append(geometry.CameraView(i, 48, 40, 40.0, 40.0, 23.5, 19.5, rr, tt))
    images = [d[f"img{i}"] for i in range(3)]
    for workers in (2, 3):
        sc = scene_m.build_hierarchy(tpts, 0.25, 2, offsets_per_voxel=3, seed=4, views=views)
        cfg = trainer.TrainConfig(total_steps=8, batch_size=3, workers=workers, step2_start=8,
                                  step3_start=8, growth_stop=0, log_every=0)
        st = trainer.make_state(sc, cfg)
        reps = [trainer.train_step(st, views, images) for _ in range(2)]
        out[f"w{workers}_transfer"] = np.array([r_.transfer_bytes for r_ in reps])
        out[f"w{workers}_rgb"] = np.array([r_.rgb for r_ in reps])
    np.savez_compressed(OUT / "boundary.npz", **out)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    which = sys.argv[1:] or ["scene_small", "raster_leaf", "train_small", "cfg1", "depth_prior",
                             "geo_loss"]
    for name in which:
        t0 = time.time()
        globals()[f"make_{name}"]()
        print(f"{name}: {time.time() - t0:.1f}s")
