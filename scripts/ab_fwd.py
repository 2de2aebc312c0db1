"""Run one view's compositor forward with library builds given as VSX_LIB
paths ("base" = the in-tree build) in subprocesses and check that every
output plane is bit-identical (the forward has no atomics)."""
import os, subprocess, sys
import numpy as np

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2503_23044_b200 import device as D
from paper_2503_23044_b200.trainer import TrainConfig, TrainState
scene, views, desc, _ = bench.workload("cfg2")
st = TrainState(scene, TrainConfig(total_steps=100, step2_start=100, step3_start=100, growth_stop=0))
ds = st.dscene
status = torch.zeros(1, dtype=torch.int32, device="cuda")
out = {}
for vi in (0, 3):
    v = views[vi]
    act = ds.active(v)
    dec = D.decode(st.params.abi(), st.n, act, ds.centers, st.anchors.emb, st.anchors.log_scales, st.anchors.offsets, v, ds.lod_ref, ds.max_scale, status, keep_cache=False)
    P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, v, status)
    B = D.bin_tiles(P, v.width, v.height)
    R = D.raster_forward(P, B, v)
    for k in ("rgb", "alpha", "depth", "normal", "raw_normal", "t_final", "n_contrib"):
        t = getattr(R, k, None)
        if t is not None:
            out[f"{vi}_{k}"] = t.cpu().numpy()
np.savez(sys.argv[1], **out)
'''

outs = []
for i, lib in enumerate(sys.argv[1:]):
    env = dict(os.environ)
    env.pop("VSX_LIB", None)
    if lib != "base":
        env["VSX_LIB"] = lib
    path = f"/tmp/fwd_{i}.npz"
    subprocess.run([sys.executable, "-c", CHILD, path], check=True, env=env)
    outs.append((lib, np.load(path)))
base_name, base = outs[0]
ok = True
for name, o in outs[1:]:
    for k in base.files:
        same = np.array_equal(base[k], o[k])
        ok &= same
        if not same:
            print(f"{name}: {k} differs, max abs {np.abs(base[k].astype(np.float64) - o[k]).max()}")
    print(f"{name} vs {base_name}: {'bit-identical' if ok else 'DIFFERENT'} over {len(base.files)} planes")
sys.exit(0 if ok else 1)
