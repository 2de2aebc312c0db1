"""Backward work per view: sum over tiles of 256 * max(n_contrib) (what the
chunked backward walks) vs sum over pixels of n_contrib (live pairs)."""
import sys, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2503_23044_b200 import device as D
from paper_2503_23044_b200.trainer import TrainConfig, TrainState
scene, views, desc, _ = bench.workload("cfg2")
st = TrainState(scene, TrainConfig(total_steps=100, step2_start=100, step3_start=100, growth_stop=0))
ds = st.dscene
status = torch.zeros(1, dtype=torch.int32, device="cuda")
for v in views[:3]:
    act = ds.active(v)
    dec = D.decode(st.params.abi(), st.n, act, ds.centers, st.anchors.emb, st.anchors.log_scales, st.anchors.offsets, v, ds.lod_ref, ds.max_scale, status, keep_cache=False)
    P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, v, status)
    B = D.bin_tiles(P, v.width, v.height)
    R = D.raster_forward(P, B, v)
    nc = R.n_contrib.view(v.height, v.width).long()
    H, W = v.height, v.width
    pad = torch.zeros((B.tiles_y * 16, B.tiles_x * 16), dtype=torch.long, device="cuda")
    pad[:H, :W] = nc
    t = pad.view(B.tiles_y, 16, B.tiles_x, 16).permute(0, 2, 1, 3).reshape(-1, 256)
    smax = t.max(dim=1).values
    chunks16 = ((smax + 15) // 16) * 16
    lists = torch.diff(B.tile_offsets.long())
    print(f"view {v.view_id}: live {nc.sum().item()/1e6:.0f}M  walked(256*smax) {(256*smax).sum().item()/1e6:.0f}M  "
          f"walked16 {(256*chunks16).sum().item()/1e6:.0f}M  list {256*lists.sum().item()/1e6:.0f}M  "
          f"mean nc {nc.float().mean().item():.1f} mean smax {smax.float().mean().item():.1f} mean list {lists.float().mean().item():.1f}", flush=True)
