"""Fraction of (tile, splat) bin entries whose alpha is below a threshold at
every pixel of the tile (exact zero = the exp2 underflows for all 256 pixels)."""
import math, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2503_23044_b200 import device as D
from paper_2503_23044_b200.trainer import TrainConfig, TrainState
scene, views, desc, _ = bench.workload("cfg2")
st = TrainState(scene, TrainConfig(total_steps=100, step2_start=100, step3_start=100, growth_stop=0))
ds = st.dscene
status = torch.zeros(1, dtype=torch.int32, device="cuda")
L2E = 1.4426950408889634
for v in views[:3]:
    act = ds.active(v)
    dec = D.decode(st.params.abi(), st.n, act, ds.centers, st.anchors.emb, st.anchors.log_scales, st.anchors.offsets, v, ds.lod_ref, ds.max_scale, status, keep_cache=False)
    P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, v, status)
    B = D.bin_tiles(P, v.width, v.height)
    rec = P.rec[: P.count]
    m = rec[:, :4].contiguous().view(torch.float64)          # mean2d
    conic, op = rec[:, 4:7], rec[:, 7]
    off = B.tile_offsets.long()
    T = off.numel() - 1
    tile_of = torch.repeat_interleave(torch.arange(T, device="cuda"), torch.diff(off))
    lst = B.tile_list.long()
    ox = (tile_of % B.tiles_x).double() * 16; oy = (tile_of // B.tiles_x).double() * 16
    mx = (m[lst, 0] - ox).float(); my = (m[lst, 1] - oy).float()
    a = -0.5 * L2E * conic[lst, 0]; b = -L2E * conic[lst, 1]; c = -0.5 * L2E * conic[lst, 2]
    o = op[lst]
    best = torch.full_like(mx, -1e30)
    pix = torch.arange(16, device="cuda", dtype=torch.float32)
    for ly in range(16):
        dy = pix.new_full((1,), float(ly)) - my[:, None]          # (I,1)
        dx = pix[None, :] - mx[:, None]                             # (I,16)
        p2 = (a[:, None] * dx + b[:, None] * dy) * dx + (c[:, None] * dy) * dy
        best = torch.maximum(best, p2.max(dim=1).values)
    amax = o * torch.exp2(torch.clamp(best, max=0.0))
    n = lst.numel()
    print(f"view {v.view_id}: entries {n}  exact-zero {(best < -126).float().mean().item():.3f}  "
          f"<1e-6 {(amax < 1e-6).float().mean().item():.3f}  <1e-4 {(amax < 1e-4).float().mean().item():.3f}  "
          f"<1/255 {(amax < 1/255).float().mean().item():.3f}", flush=True)
