"""Work model of the compositor backward on one cfg2 view (GPU box): listed
pairs (256 x list length), the pairs the chunk loop visits (256 x max live
count per tile), the live-prefix pairs (slots sorted by live count >> 3) and
the live pairs (sum of per-pixel live counts)."""
import sys
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import test_gpu_parity_scale as T  # noqa: E402
from paper_2503_23044_b200 import _lib, device as D  # noqa: E402
_lib.load()

c = T.build_cfg2_view()
P, B, view = c["P"], c["B"], c["view"]
R = D.raster_forward(P, B, view)
H, W = view.height, view.width
nc = R.n_contrib.cpu().numpy().reshape(H, W)
off = B.tile_offsets.long().cpu().numpy()
tx, ty = (W + 15) // 16, (H + 15) // 16
pad = np.zeros((ty * 16, tx * 16), np.int64)
pad[:H, :W] = nc
tiles = pad.reshape(ty, 16, tx, 16).transpose(0, 2, 1, 3).reshape(ty * tx, 256)
lens = off[1:] - off[:-1]
smax = tiles.max(1)
listed = 256 * lens.sum()
visited = 256 * smax.sum()
live = tiles.sum()
# chunks of 16 from s_max down; prefix = slots with (nc >> 3) >= (kbase >> 3), rounded to 8
pref = 0
warp_work = 0
for t in range(len(smax)):
    s = int(smax[t])
    if s == 0:
        continue
    b = np.minimum(tiles[t] >> 3, 255)
    srt = np.sort(tiles[t])[::-1]
    ce = s
    while ce > 0:
        cs = max(ce - 16, 0)
        n = int((b >= min(cs >> 3, 255)).sum())
        pref += 8 * ((n + 7) // 8) * (ce - cs)
        # phase-1 work of the sorted warps: per warp max live count in the chunk
        jl = np.clip(srt - cs, 0, ce - cs).reshape(8, 32).max(1)
        warp_work += 32 * jl.sum()
        ce = cs
print(f"tiles {len(smax)}  intersections {lens.sum()}")
print(f"listed pairs  {listed / 1e6:9.1f} M")
print(f"visited pairs {visited / 1e6:9.1f} M  ({visited / listed:.3f} of listed)")
print(f"prefix pairs  {pref / 1e6:9.1f} M  ({pref / visited:.3f} of visited)")
print(f"phase-1 warp pairs (sorted) {warp_work / 1e6:9.1f} M  ({warp_work / visited:.3f})")
print(f"live pairs    {live / 1e6:9.1f} M  ({live / visited:.3f} of visited)")
q = np.quantile(smax[smax > 0], [0.5, 0.9, 0.99, 1.0])
print("s_max quantiles 50/90/99/100:", q)
