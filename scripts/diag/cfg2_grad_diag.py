"""Diagnose cfg2 sampled-tile per-splat gradient mismatches (GPU box).

Runs the two cfg2 tests of tests/test_gpu_parity_scale.py with the final
comparison replaced by a report of the worst elements."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import test_gpu_parity_scale as T  # noqa: E402
from gpu_util import noise_floor_close  # noqa: E402
from paper_2503_23044_b200 import _lib  # noqa: E402
_lib.load()

CTX = {}


def diag(dev, leaves, touched, what):
    B = CTX["c"]["B"]
    off = B.tile_offsets.long().cpu().numpy()
    lst = B.tile_list.long().cpu().numpy()
    tile_of = {}
    for t in CTX["tiles"]:
        for s in lst[off[t]:off[t + 1]]:
            tile_of.setdefault(int(s), []).append((int(t), int(off[t + 1] - off[t]),
                                                   int(np.searchsorted(lst[off[t]:off[t + 1]], s))))
    print(f"=== {what}: touched {touched.sum()} splats")
    for name, a, b in T.GRAD_COLS:
        ref = leaves[name].grad
        ref = np.zeros((dev.shape[0], b - a)) if ref is None else ref.numpy().reshape(dev.shape[0], -1)
        got = dev[:, a:b]
        r, g = ref[touched], got[touched]
        rms = np.sqrt(np.mean(r * r))
        for noise in (1e-3, 1e-4, 1e-5):
            ok, w, ex = noise_floor_close(g, r, 1e-3, noise)
            print(f"  {name}: noise {noise:g}: worst {w:.3g} excluded {ex}")
        rel = np.abs(g - r) / np.maximum(np.abs(r), 1e-300)
        keep = np.abs(r) >= 1e-3 * rms
        rel[~keep] = 0
        idx = np.argsort(rel.ravel())[-5:]
        sidx = np.flatnonzero(touched)
        for i in idx[::-1]:
            row, col = divmod(int(i), r.shape[1])
            s = int(sidx[row])
            print(f"    splat {s} col {col}: ref {r[row, col]:.6g} got {g[row, col]:.6g} "
                  f"|ref|/rms {abs(r[row, col]) / rms:.3g} rel {rel.ravel()[i]:.3g} tiles {tile_of.get(s)}")
        big = np.abs(r).max(axis=1)
        print(f"    rms {rms:.3g} max {np.abs(r).max():.3g}")


T._compare_splat_grads = diag
c = T.build_cfg2_view()
CTX["c"] = c
tiles, lens = T._sample_tiles(c["B"])
CTX["tiles"] = tiles
print("tiles", tiles.size, "max len", lens.max(), "mean", lens[lens > 0].mean())
for fn in (T.test_cfg2_sampled_tiles_forward_and_backward_vs_oracle,
           T.test_cfg2_sampled_tiles_fused_objective_vs_oracle):
    try:
        fn(c)
    except AssertionError as e:
        print("ASSERT", fn.__name__, e)
