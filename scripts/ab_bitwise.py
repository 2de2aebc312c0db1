"""Run one view's compositor backward with two library builds (VSX_LIB A/B)
in subprocesses and compare the per-splat gradients (float atomics make
repeated runs differ in the last bits, so compare against base-vs-base)."""
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
v = views[0]
act = ds.active(v)
dec = D.decode(st.params.abi(), st.n, act, ds.centers, st.anchors.emb, st.anchors.log_scales, st.anchors.offsets, v, ds.lod_ref, ds.max_scale, status, keep_cache=False)
P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, v, status)
B = D.bin_tiles(P, v.width, v.height)
R = D.raster_forward(P, B, v)
g = torch.Generator(device="cuda").manual_seed(0)
cot = {k: torch.randn(t.shape, device="cuda", generator=g) for k, t in
       (("rgb", R.rgb), ("alpha", R.alpha), ("depth", R.depth), ("normal", R.normal))}
gs = D.raster_backward(P, B, v, R, g_rgb=cot["rgb"], g_alpha=cot["alpha"], g_depth=cot["depth"],
                       g_normal=cot["normal"])
np.save(sys.argv[1], gs.cpu().numpy())
'''


def run(lib, out):
    env = dict(os.environ)
    if lib:
        env["VSX_LIB"] = lib
    else:
        env.pop("VSX_LIB", None)
    subprocess.run([sys.executable, "-c", CHILD, out], check=True, env=env)


def compare(x, y, what):
    ga, gb = np.load(x).astype(np.float64), np.load(y).astype(np.float64)
    rel = np.linalg.norm(ga - gb, axis=0) / (np.linalg.norm(ga, axis=0) + 1e-300)
    print(what, "bitwise-identical fraction %.4f" % (ga == gb).mean(),
          "per-feature rel L2", np.array2string(rel, precision=2))


a, b = sys.argv[1], sys.argv[2]
run(None if a == "base" else a, "/tmp/ga.npy")
run(None if a == "base" else a, "/tmp/ga2.npy")
run(None if b == "base" else b, "/tmp/gb.npy")
compare("/tmp/ga.npy", "/tmp/ga2.npy", "A vs A:")
compare("/tmp/ga.npy", "/tmp/gb.npy", "A vs B:")
