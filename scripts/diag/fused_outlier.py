"""Per-tile breakdown of the worst element of the fused-objective cfg2 test
(GPU box): which sampled tile's contribution differs from the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import test_gpu_parity_scale as T  # noqa: E402
import oracle  # noqa: E402
from paper_2503_23044_b200 import _lib, device as D  # noqa: E402
from paper_2503_23044_b200._lib import VsxLossDesc  # noqa: E402
_lib.load()
SPLAT, COL = int(sys.argv[1]) if len(sys.argv) > 1 else 90804, 1

c = T.build_cfg2_view()
P, B, view = c["P"], c["B"], c["view"]
tiles, _ = T._sample_tiles(B)
H, W = view.height, view.width
off = B.tile_offsets.long().cpu().numpy()
lst = B.tile_list.long().cpu().numpy()
mine = [int(t) for t in tiles if SPLAT in set(lst[off[t]:off[t + 1]].tolist())]
print("tiles containing splat", SPLAT, mine)
R0 = D.raster_forward(P, B, view)
guard = T._guard_ok(R0, view, margin=1e-2)
rng = np.random.default_rng(8)
m = T._tile_mask(view, tiles)


def away(x, lo, hi):
    sgn = np.where(rng.uniform(size=x.shape) < 0.5, -1.0, 1.0)
    return (x + sgn * rng.uniform(lo, hi, x.shape)).astype(np.float32)


rgb0 = R0.rgb.cpu().numpy()
gt = np.where(m[..., None], away(rgb0, 0.01, 0.5), rgb0)
d0 = R0.depth.cpu().numpy()
pdep = (d0 * (1.0 + away(np.zeros_like(d0), 0.01, 0.1))).astype(np.float32)
pv = (m & guard & (rng.uniform(size=(H, W)) > 0.2)).astype(np.uint8)
pn = away(R0.normal.cpu().numpy(), 0.01, 0.5)
pnv = (m & guard & (rng.uniform(size=(H, W)) > 0.3)).astype(np.uint8)
leaves = T._device_leaves(P)
for t in mine:
    # objective restricted to this one tile: targets equal the render elsewhere
    mt = T._tile_mask(view, [t])
    g1 = np.where(mt[..., None], gt, rgb0)
    pv1 = (pv & mt).astype(np.uint8)
    pnv1 = (pnv & mt).astype(np.uint8)
    dt = {k: torch.as_tensor(v).cuda() for k, v in
          (("gt", g1), ("pd", pdep), ("pv", pv1), ("pn", pn), ("pnv", pnv1))}
    sums = torch.zeros(3, dtype=torch.float64, device="cuda")
    counts = torch.zeros(2, dtype=torch.int32, device="cuda")
    live = torch.zeros((), dtype=torch.int64, device="cuda")
    loss = VsxLossDesc(gt_rgb=dt["gt"].data_ptr(), prior_depth=dt["pd"].data_ptr(),
                       prior_depth_valid=dt["pv"].data_ptr(), prior_normal=dt["pn"].data_ptr(),
                       prior_normal_valid=dt["pnv"].data_ptr(), rgb_scale=1.0 / (H * W * 3),
                       depth_weight=1.0, normal_weight=0.5 / 3.0, sums=sums.data_ptr(),
                       counts=counts.data_ptr(), live_pairs=live.data_ptr())
    R = D.raster_forward(P, B, view, loss=loss)
    dev = D.raster_backward(P, B, view, R, loss=loss).double().cpu().numpy()
    cnt = counts.cpu().numpy()
    for k in leaves.values():
        k.grad = None
    outs = T._oracle_tiles(leaves, B, [t], view)
    o, ins, py, px = outs[0]
    ki = torch.from_numpy(ins)
    gt_t = torch.from_numpy(g1.astype(np.float64))
    pd_t = torch.from_numpy(pdep.astype(np.float64))
    pn_t = torch.from_numpy(pn.astype(np.float64))
    pvb, pnvb = torch.from_numpy(pv1.astype(bool)), torch.from_numpy(pnv1.astype(bool))
    rgb_s = (o["rgb"][ki] - gt_t[py, px]).abs().sum()
    md = (o["valid"][ki] & pvb[py, px]).double()
    dep_s = ((o["depth"][ki] - pd_t[py, px]).abs() * md).sum()
    mn = (o["valid"][ki] & pnvb[py, px]).double()
    nrm_s = ((o["normal"][ki] - pn_t[py, px]).abs().sum(-1) * mn).sum()
    obj = rgb_s / (H * W * 3) + dep_s / max(int(cnt[0]), 1) + 0.5 * nrm_s / (3.0 * max(int(cnt[1]), 1))
    obj.backward()
    ref = leaves["mean2d"].grad[SPLAT].numpy()
    got = dev[SPLAT, 0:2]
    j = int(np.searchsorted(lst[off[t]:off[t + 1]], SPLAT))
    print(f"tile {t} len {off[t+1]-off[t]} pos {j} counts {cnt.tolist()}: ref {ref} got {got} "
          f"rel {np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)}")
    ncs = R.n_contrib.cpu().numpy()[py, px]
    print("   n_contrib min/median/max", ncs.min(), np.median(ncs), ncs.max(),
          "pixels with depth prior", int(md.sum()), "normal prior", int(mn.sum()))
    # which pixel terms dominate: per-pixel oracle contributions of this splat
rec = P.rec.cpu()
print("splat record", rec[SPLAT, :8].tolist(), "mean2d", rec.view(torch.float64)[SPLAT, :2].tolist())
