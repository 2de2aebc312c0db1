"""The reference CPU arm of bench.py (TEST INFRASTRUCTURE ONLY).

Drives the UNMODIFIED reference package installed in ``oracle/_ref`` by
``oracle/build_ref.py`` (``/root/reference/pkg``, float64 CPU) through its
own public API; nothing here re-implements the reference's math.

* :func:`cfg1_step_seconds` — one full ``voxsplat.trainer.train_step`` at
  SURVEY §8(d) cfg1 (10,198 anchors x 10, 4 views at 128^2, RGB loss), the
  CPU-runnable config, at a given torch thread count.
* :class:`Cfg2Sampler` — a bounded sample of the bench workload (cfg2:
  ~200k anchors x 10, 8 views at 1920x1080, RGB + Eq. 9 depth + normal prior
  loss) per call, since the reference's padded (T, L, 256) float64
  compositor cannot hold a full 1080p view (SURVEY §7 hard part 8). One call
  runs, for one view: the reference's ``transfer_gaussians`` (cull + decode,
  graph kept) + ``project_splats`` + ``bin_splats`` in full; its
  ``rasterize_patch`` forward + autograd backward on an evenly spaced
  sample of the view's non-empty 16x16 tiles (scaled up by intersections);
  the autograd backward through projection and decode for the whole view;
  and the reference's Adam (``apply_decoder_grads`` / ``apply_level_grads``)
  over every parameter once per step. The normal-prior term is the
  reference's own ``e_depth_loss`` per normal channel (the contract pinned
  in ``tests/golden/normal_prior.npz``).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np
import torch

REF_DIR = Path(__file__).resolve().parent / "_ref"


def load_reference():
    """Import voxsplat from oracle/_ref (raises if the recipe was not run)."""
    if not (REF_DIR / "voxsplat" / "__init__.py").exists():
        raise ImportError("oracle/_ref not installed: run `python oracle/build_ref.py` "
                          "(or __graft_entry__.build()) where /root/reference exists")
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import voxsplat
    if Path(voxsplat.__file__).resolve().parent.parent != REF_DIR.resolve():
        raise ImportError(f"voxsplat resolved to {voxsplat.__file__}, not oracle/_ref")
    from voxsplat import geometry, losses, partition, renderer, scene, trainer
    return {"geometry": geometry, "losses": losses, "partition": partition,
            "renderer": renderer, "scene": scene, "trainer": trainer}


def _ref_view(ref, v):
    return ref["geometry"].CameraView(int(v.view_id), int(v.width), int(v.height), float(v.fx),
                                      float(v.fy), float(v.cx), float(v.cy),
                                      np.asarray(v.r, np.float64), np.asarray(v.t, np.float64))


def cfg1_step_seconds(threads: int) -> dict:
    """One reference train_step at cfg1 (the survey recipe) with `threads` threads."""
    ref = load_reference()
    old = torch.get_num_threads()
    torch.set_num_threads(threads)
    try:
        sc, geo, tr = ref["scene"], ref["geometry"], ref["trainer"]
        rng = np.random.default_rng(0)
        pts = np.stack([rng.uniform(-1, 1, 120000), rng.uniform(-1, 1, 120000),
                        rng.uniform(-0.005, 0.005, 120000)], -1)
        scene = sc.build_hierarchy(sc.SparsePoints(pts), base_voxel_size=0.02, lod_count=1,
                                   offsets_per_voxel=10, seed=0)
        f = 64.0 / np.tan(np.radians(30.0))
        views = []
        for i in range(4):
            eye = np.array([0.3 * np.cos(np.pi * i / 2), 0.3 * np.sin(np.pi * i / 2), 2.2])
            r, t = geo.look_at(eye, np.zeros(3), up=(0.0, 1.0, 0.0))
            views.append(geo.CameraView(i, 128, 128, f, f, 63.5, 63.5, r, t))
        scene.set_lod_reference(views)
        images = [rng.uniform(0, 1, (128, 128, 3)) for _ in range(4)]
        cfg = tr.TrainConfig(total_steps=100, batch_size=4, workers=1, step2_start=100,
                             step3_start=100, growth_stop=0, log_every=0)
        state = tr.make_state(scene, cfg)
        t0 = time.perf_counter()
        rep = tr.train_step(state, views, images)
        sec = time.perf_counter() - t0
    finally:
        torch.set_num_threads(old)
    return {"seconds": sec, "views": 4, "views_per_s": 4 / sec, "threads": threads,
            "rgb_loss": rep.rgb}


class Cfg2Sampler:
    """Bounded per-call samples of one training step of the bench workload.

    Setup runs, for ``front_views`` views of the batch, the reference's front
    end (``transfer_gaussians`` with the graph kept, ``project_splats``,
    ``bin_splats``) and one autograd pass from the projected splats back to
    the decoder / anchor leaves (random cotangents, graph retained), timing
    each: those are the per-view fixed costs (~6% of a cfg2 view). Every
    call then composites a fresh, evenly spaced sample of the view's
    non-empty tiles exactly as the reference's ``rasterize_view`` does — the
    tiles grouped into its next-power-of-two length buckets, one
    ``_blend_padded`` + ``_finalize`` per bucket (renderer.py:390-449) — with
    the RGB + Eq. 9 depth + normal-prior loss on those pixels, back-propagates
    it to the splat tensors, and runs the reference's Adam over every
    parameter. A view's time = front + proj/decode backward + composite
    fwd+bwd x (view intersections / sampled intersections); a step = B views
    + one Adam.
    """

    def __init__(self, points, base_voxel_size: float, lod_count: int, lod_bias: int, n: int,
                 views, tiles: int, normal_weight: float = 0.5, seed: int = 0,
                 front_views: int = 2):
        ref = self.ref = load_reference()
        sc, tr = ref["scene"], ref["trainer"]
        self.views = [_ref_view(ref, v) for v in views]
        scene = sc.build_hierarchy(sc.SparsePoints(np.asarray(points, np.float64)),
                                   base_voxel_size, lod_count, offsets_per_voxel=n, seed=seed,
                                   views=self.views)
        scene.lod_bias = lod_bias
        self.scene = scene
        B = len(views)
        self.cfg = tr.TrainConfig(total_steps=30000, batch_size=B, workers=1, step2_start=0,
                                  step3_start=30000, growth_stop=0, log_every=0)
        self.state = tr.make_state(scene, self.cfg)
        self.tiles = int(tiles)
        self.normal_weight = float(normal_weight)
        rng = np.random.default_rng(seed + 1)
        self.targets = []
        for v in self.views:
            H, W = v.height, v.width
            nrm = rng.normal(size=(H, W, 3))
            self.targets.append({
                "rgb": torch.as_tensor(rng.uniform(0, 1, (H, W, 3))),
                "depth": rng.uniform(20.0, 60.0, (H, W)), "dvalid": rng.uniform(size=(H, W)) > 0.1,
                "normal": nrm / np.linalg.norm(nrm, axis=-1, keepdims=True),
                "nvalid": rng.uniform(size=(H, W)) > 0.1})
        self.fronts = [self._front(i) for i in range(min(front_views, B))]
        self.calls = 0

    KEYS = ("mean2d", "conic", "color", "opacity", "normal_cam", "plane_d")

    def _front(self, vi: int) -> dict:
        R, st = self.ref["renderer"], self.state
        view = self.views[vi]
        t0 = time.perf_counter()
        batch, _ = R.transfer_gaussians(view, st.scene, st.assignment, st.replicas[0],
                                        state=st.decode_state(), keep_graph=True)
        splats = R.project_splats(batch, view)
        lists = R.bin_splats(splats, view.width, view.height)
        t1 = time.perf_counter()
        dec = st.replicas[0].tensors
        level_keys = [(k, key) for k in sorted(st.level_state)
                      for key in ("embeddings", "log_scales", "offsets")]
        inputs = [dec[n] for n in dec] + [st.level_state[k][key] for k, key in level_keys]
        outs = [getattr(splats, k) for k in self.KEYS]
        gen = torch.Generator().manual_seed(vi)
        cots = [torch.randn(o.shape, generator=gen, dtype=o.dtype) for o in outs]
        t2 = time.perf_counter()
        grads = torch.autograd.grad(outs, inputs, grad_outputs=cots, allow_unused=True,
                                    retain_graph=True)
        t3 = time.perf_counter()
        counts = np.array([len(x) for x in lists])
        return {"vi": vi, "splats": splats, "lists": lists, "counts": counts,
                "busy": np.flatnonzero(counts > 0), "front_s": t1 - t0, "bwd_s": t3 - t2,
                "grads": grads, "names": list(dec), "level_keys": level_keys,
                "gaussians": int(batch.count)}

    def sample(self) -> dict:
        """One bounded sample plus one Adam; returns timings and the
        extrapolated views/s of a full B-view step."""
        ref, st = self.ref, self.state
        R, L = ref["renderer"], ref["losses"]
        B = len(self.views)
        f = self.fronts[self.calls % len(self.fronts)]
        rot = self.calls // len(self.fronts)
        self.calls += 1
        view, tg = self.views[f["vi"]], self.targets[f["vi"]]
        H, W = view.height, view.width
        splats, lists, counts, busy = f["splats"], f["lists"], f["counts"], f["busy"]
        k = min(self.tiles, busy.size)
        stride = busy.size / max(k, 1)
        pick = busy[((np.arange(k) + 0.37 * (rot % 7)) * stride).astype(np.int64) % busy.size]
        pick = np.unique(pick)
        pix_u, pix_v, in_img = R._tile_pixel_grids(W, H)
        leaves = {key: getattr(splats, key).detach().clone().requires_grad_(True)
                  for key in self.KEYS}
        real = {key: getattr(splats, key) for key in self.KEYS}
        t0 = time.perf_counter()
        for key in self.KEYS:
            setattr(splats, key, leaves[key])
        try:
            obj = torch.zeros((), dtype=torch.float64)
            plen = np.int64(1) << np.int64(np.ceil(np.log2(counts[pick]))).clip(min=0)
            for size in np.unique(plen):
                rows = pick[plen == size]
                idx_mat = np.zeros((rows.size, int(size)), dtype=np.int64)
                pad = np.zeros((rows.size, int(size)), dtype=bool)
                for row, t in enumerate(rows):
                    idx_mat[row, :lists[t].size] = lists[t]
                    pad[row, :lists[t].size] = True
                raw = R._blend_padded(splats, idx_mat, pad, torch.from_numpy(pix_u[rows]),
                                      torch.from_numpy(pix_v[rows]), view, R.ALL_TASKS)
                fin, valid = R._finalize(raw, R.ALL_TASKS)
                keep = torch.from_numpy(in_img[rows])
                py = torch.from_numpy(pix_v[rows].astype(np.int64))[keep]
                px = torch.from_numpy(pix_u[rows].astype(np.int64))[keep]
                obj = obj + L.bl_rgb_loss([fin["rgb"][keep]], [tg["rgb"][py, px]]) / B
                d_loss, _ = L.e_depth_loss([fin["depth"][keep]], [valid[keep]],
                                           [tg["depth"][py.numpy(), px.numpy()]],
                                           [tg["dvalid"][py.numpy(), px.numpy()]])
                obj = obj + d_loss / B
                for c in range(3):
                    n_loss, _ = L.e_depth_loss(
                        [fin["normal"][keep][:, c]], [valid[keep]],
                        [tg["normal"][py.numpy(), px.numpy(), c]],
                        [tg["nvalid"][py.numpy(), px.numpy()]])
                    obj = obj + self.normal_weight / 3.0 * n_loss / B
            t1 = time.perf_counter()
            gl = torch.autograd.grad(obj, [leaves[key] for key in self.KEYS],
                                     allow_unused=True) if obj.requires_grad else None
            t2 = time.perf_counter()
        finally:
            for key in self.KEYS:
                setattr(splats, key, real[key])
        del gl
        names, level_keys, grads = f["names"], f["level_keys"], f["grads"]
        dec = st.replicas[0].tensors
        t3 = time.perf_counter()
        st.apply_decoder_grads({nm: (g if g is not None else torch.zeros_like(dec[nm]))
                                for nm, g in zip(names, grads[:len(names)])})
        lg: dict = {}
        for (lv, key), g in zip(level_keys, grads[len(names):]):
            lg.setdefault(lv, {})[key] = g if g is not None else \
                torch.zeros_like(st.level_state[lv][key])
        for lv in sorted(lg):
            st.apply_level_grads(lv, lg[lv])
        t4 = time.perf_counter()
        isect_total = int(counts.sum())
        isect_sampled = int(counts[pick].sum())
        scale = isect_total / max(isect_sampled, 1)
        view_s = f["front_s"] + f["bwd_s"] + (t2 - t0) * scale
        step_s = B * view_s + (t4 - t3)
        return {"views_per_s": B / step_s, "step_s": step_s, "view_s": view_s,
                "front_s": f["front_s"], "proj_decode_bwd_s": f["bwd_s"],
                "tiles_fwd_s": t1 - t0, "tiles_bwd_s": t2 - t1, "adam_s": t4 - t3,
                "wall_s": (t2 - t0) + (t4 - t3), "tiles": int(pick.size),
                "tiles_nonempty": int(busy.size), "isect_sampled": isect_sampled,
                "isect_total": isect_total, "gaussians": f["gaussians"], "view": f["vi"]}
