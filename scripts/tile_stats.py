import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2503_23044_b200 import device as D
from paper_2503_23044_b200.trainer import TrainConfig, TrainState
scene, views, desc, _ = bench.workload("cfg2")
st = TrainState(scene, TrainConfig(total_steps=100, step2_start=100, step3_start=100, growth_stop=0))
ds = st.dscene
status = torch.zeros(1, dtype=torch.int32, device="cuda")
for v in views[:4]:
    act = ds.active(v)
    dec = D.decode(st.params.abi(), st.n, act, ds.centers, st.anchors.emb, st.anchors.log_scales, st.anchors.offsets, v, ds.lod_ref, ds.max_scale, status, keep_cache=False)
    P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, v, status)
    Bn = D.bin_tiles(P, v.width, v.height)
    c = torch.diff(Bn.tile_offsets.long()).cpu().numpy()
    print(Bn.intersections, c.max(), np.percentile(c, [50, 90, 99, 99.9]), (c > 4096).sum(), (c > 8192).sum(), c[c>4096].sum()/c.sum())
