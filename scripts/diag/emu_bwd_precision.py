"""Where the fp32 error of the per-splat 2D gradients comes from (CPU only).

Builds view 0 of the cfg2 workload with the float64 oracle (decode, project,
bin), then for heavy tiles emulates the compositing forward + backward of
the CUDA kernels in float32 numpy with random pixel cotangents and compares
per-splat gradients with the oracle's float64 autograd:

  f32     every step float32 (T recovered back to front by division);
  Texact  the backward uses the forward's own float32 T (no division chain);
  all64   the backward entirely in float64 on the float32 forward's alphas.

Worst relative error over elements with |g| >= EPS * rms(g) of their column
(EPS from argv, default 1e-3). Measured: all64 is no better than f32, i.e.
the residual is the float32 rounding of the forward's alpha / T, not the
backward arithmetic; at EPS = 1e-2 every variant is <= ~4e-4.

  python scripts/diag/emu_bwd_precision.py [EPS]
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402


def _cfg2_view0():
    import bench
    scene, views, _desc, _ = bench.workload("cfg2")
    n = scene.offsets_per_voxel
    w = oracle.decoder_init(n, 0, float(np.log(0.125 * scene.base_voxel_size)))
    f32r = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    st = oracle.OracleState.create(
        scene.flat_centers(), scene.flat_levels(), scene.lod_count, scene.lod_ref_distance,
        scene.lod_bias, scene.base_voxel_size, n, {k: f32r(v) for k, v in w.items()},
        f32r(scene.flat("embeddings")), f32r(np.log(scene.flat("scales"))),
        f32r(scene.flat("offsets")))
    cam = oracle.Cam.of(views[0])
    with torch.no_grad():
        P, _, _ = oracle.pipeline._view_splats(st, cam, grad=False)
    off, lst = oracle.bin_tiles(P["mean2d"].numpy(), P["radius"], cam.width, cam.height)
    out = {k: P[k].numpy() for k in oracle.SPLAT_KEYS}
    out.update(off=off, lst=lst, fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, W=cam.width,
               H=cam.height)
    return out


d = _cfg2_view0()
off, lst = d["off"], d["lst"]
lens = np.diff(off)
W, H = int(d["W"]), int(d["H"])
txn = (W + 15) // 16
cam = oracle.Cam(np.eye(3), np.zeros(3), np.zeros(3), float(d["fx"]), float(d["fy"]), float(d["cx"]), float(d["cy"]), W, H)
S64 = {k: torch.tensor(d[k]) for k in oracle.SPLAT_KEYS}
f32 = np.float32

def emulate(idx, tx, ty, cot, mode):
    # cot: dict of per-pixel cotangents (256,) arrays in f32 pixel order p = ly*16+lx
    m = d["mean2d"][idx]; con = d["conic"][idx].astype(f32); op = d["opacity"][idx].astype(f32)
    col = d["color"][idx].astype(f32); nrm = d["normal_cam"][idx].astype(f32); pd = d["plane_d"][idx].astype(f32)
    ox, oy = tx * 16.0, ty * 16.0
    mx = (m[:, 0] - ox).astype(f32); my = (m[:, 1] - oy).astype(f32)
    lx = (np.arange(256) % 16).astype(f32); ly = (np.arange(256) // 16).astype(f32)
    L = len(idx)
    # alpha per (splat, pixel) in f32
    dx = lx[None, :] - mx[:, None]; dy = ly[None, :] - my[:, None]
    pw = f32(-0.5) * (con[:, 0:1] * dx * dx + f32(2) * con[:, 1:2] * dx * dy + con[:, 2:3] * dy * dy)
    e = np.exp(np.minimum(pw, 0).astype(np.float64)).astype(f32)
    at = (op[:, None] * e).astype(f32)
    al = np.minimum(at, f32(0.99))
    # forward: T product f32, live
    T = np.ones(256, f32); Tprev = np.zeros((L, 256), f32); live = np.zeros((L, 256), bool)
    for k in range(L):
        lv = T >= f32(1e-4)
        live[k] = lv
        Tprev[k] = T
        T = np.where(lv, (T * (f32(1) - al[k])).astype(f32), T)
    nc = live.sum(0)
    # per-pixel cotangent dot per splat: s_k = gA + gC.col + gR.nrm + gD*pd
    gA, gC, gR, gD = cot
    sk = (gA[None, :] + col @ gC.T + nrm @ gR.T + pd[:, None] * gD[None, :]).astype(f32)
    # backward recursion back to front
    Tb = T.copy(); S = np.zeros(256, np.float64 if mode.get("S64") else f32)
    wpl = np.zeros((L, 256), np.float64); qpl = np.zeros((L, 256), np.float64)
    for k in range(L - 1, -1, -1):
        lv = live[k]
        a = al[k]
        if mode.get("Texact"):
            Tk = Tprev[k].astype(np.float64) if mode.get("T64") else Tprev[k]
        else:
            if mode.get("T64"):
                Tk = Tb.astype(np.float64) / (1 - a.astype(np.float64))
            else:
                Tk = (Tb / (f32(1) - a)).astype(f32)
        w = a * Tk
        da = Tk * sk[k] - S / (f32(1) - a)
        S_new = S + sk[k] * w
        S = np.where(lv, S_new, S)
        Tb = np.where(lv, Tk, Tb)
        dat = np.where(at[k] <= f32(0.99), da, 0)
        wpl[k] = np.where(lv, w, 0); qpl[k] = np.where(lv, dat * e[k], 0)
    dt = np.float64 if mode.get("sum64") else f32
    wpl = wpl.astype(dt); qpl = qpl.astype(dt)
    gcol = wpl @ gC.astype(dt)
    Q1 = qpl.sum(1)
    sx = (qpl * dx.astype(dt)).sum(1); sy = (qpl * dy.astype(dt)).sum(1)
    gop = Q1  # note: dL/dop = sum q (since q = dat*e) -> opacity grad
    gm0 = op * (con[:, 0] * sx + con[:, 1] * sy)
    return {"color": gcol, "opacity": gop, "mean0": gm0}

def exact(idx, tx, ty, cot):
    leaves = {k: S64[k][torch.from_numpy(idx)].clone().requires_grad_(True) for k in oracle.SPLAT_KEYS}
    out = oracle.raster_tile(leaves, np.arange(len(idx)), tx, ty, cam)
    gA, gC, gR, gD = [torch.tensor(c.astype(np.float64)) for c in cot]
    # out["alpha"], rgb, raw_normal, dist are the blended channels
    obj = (out["alpha"] * gA).sum() + (out["rgb"] * gC).sum() + (out["raw_normal"] * gR).sum() + (out["dist"] * gD).sum()
    obj.backward()
    g = {k: leaves[k].grad.numpy() for k in oracle.SPLAT_KEYS}
    return {"color": g["color"], "opacity": g["opacity"], "mean0": g["mean2d"][:, 0]}

EPS = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
rng = np.random.default_rng(0)
heavy = np.argsort(lens)[-3:]
mid = np.flatnonzero(lens > 800)[:3]
for t in list(heavy) + list(mid):
    ty, tx = divmod(int(t), txn)
    idx = lst[off[t]:off[t + 1]]
    cot = (rng.normal(size=256).astype(f32), rng.normal(size=(256, 3)).astype(f32),
           rng.normal(size=(256, 3)).astype(f32), (rng.normal(size=256) * 1e-2).astype(f32))
    ref = exact(idx, tx, ty, cot)
    line = f"tile {t} L={len(idx)}:"
    for name, mode in (("f32", {}), ("Texact", {"Texact": 1}), 
                       ("all64", {"T64": 1, "S64": 1, "sum64": 1})):
        got = emulate(idx, tx, ty, cot, mode)
        worst = {}
        for k in ref:
            r = np.asarray(ref[k]).reshape(len(idx), -1); g = np.asarray(got[k], np.float64).reshape(len(idx), -1)
            rms = np.sqrt(np.mean(r * r))
            keep = np.abs(r) >= EPS * rms
            worst[k] = (np.abs(g - r)[keep] / np.abs(r)[keep]).max()
        line += f" | {name}: " + " ".join(f"{k}={v:.1e}" for k, v in worst.items())
    print(line, flush=True)
