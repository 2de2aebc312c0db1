"""Two ranks of the sharded CUDA step on ONE GPU, as two threads of one
process over torch's in-process "threaded" process group.

The collectives (all-to-all of splat records, reverse all-to-all of the 2D
gradients, decoder all-reduce, replica checksum) run on the host between the
threads, so no kernel ever waits on another rank's kernel (the pattern the
B200 profiling guide forbids on one GPU). Compares both ranks' losses and the
owner-merged parameters with the single-process ``train_step``. Prints one
JSON line; run by tests/test_gpu_dist.py in a subprocess (it swaps the
process-wide distributed world).
"""
import json
import sys
import threading
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist
from torch.testing._internal.distributed.multi_threaded_pg import _install_threaded_pg

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))
from conftest import golden_scene, golden_view, load_golden  # noqa: E402

from paper_2503_23044_b200.dist import (CudaShardBackend, sharded_train_step,  # noqa: E402
                                        sync_growth)
from paper_2503_23044_b200.trainer import TrainConfig, TrainState, train_step  # noqa: E402

WORLD = int(sys.argv[1]) if len(sys.argv) > 1 else 2
NV = int(sys.argv[2]) if len(sys.argv) > 2 else 3   # views; < WORLD splits views into bands
GEO = len(sys.argv) > 3 and sys.argv[3] == "geo"    # Eq. 10 NCC term from step 1 on
STEPS = 2
d = load_golden("train_small")
views = [golden_view(d, f"v{i}", i) for i in range(3)]
images = [d[f"img{i}"] for i in range(3)]
priors = [(d[f"prior{i}"], d[f"pvalid{i}"]) for i in range(3)]
priors[1] = None                      # the depth term averages over views with a prior
_rng = np.random.default_rng(5)
npri = []
for _i in range(3):
    _p = _rng.normal(size=(40, 48, 3)).astype(np.float32)
    npri.append((_p / np.linalg.norm(_p, axis=-1, keepdims=True), _rng.uniform(size=(40, 48)) > 0.3))
npri[2] = None
if NV < 3:
    # keep a view with a normal prior but no depth prior among the first NV
    views, images = views[:NV], images[:NV]
    priors = [priors[0], None][:NV]
    npri = [None, npri[1]][:NV]
cfg = dict(total_steps=8, batch_size=NV, step2_start=0, step3_start=0 if GEO else 8,
           growth_stop=0, normal_weight=0.5)

import faulthandler  # noqa: E402
faulthandler.dump_traceback_later(150, exit=True)  # a hang prints every thread's stack
torch.cuda.init()
torch._C._distributed_c10d._set_thread_isolation_mode(True)  # per-thread group registry
_install_threaded_pg()


def _device_synced(fn):
    """The threaded group reduces on whichever rank thread arrives last, on
    that thread's stream; a device-wide sync on both sides orders it after
    every rank's producer kernels (NCCL does this with stream dependencies)."""
    def call(*a, **k):
        torch.cuda.synchronize()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        return r
    return call


for _name in ("all_reduce", "all_to_all_single", "all_gather", "broadcast", "barrier"):
    setattr(dist, _name, _device_synced(getattr(dist, _name)))
store = dist.HashStore()
res, errs = {}, []


def run(rank):
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("threaded", rank=rank, world_size=WORLD, store=store)
        # one stream per rank, as one process per GPU would have: the sort /
        # scan scratch buffers are keyed by stream
        with torch.cuda.stream(torch.cuda.Stream()):
            st = TrainState(golden_scene(d), TrainConfig(**cfg, workers=WORLD))
            be = CudaShardBackend(st, rank, WORLD)
            reps = [sharded_train_step(be, views, images, priors, npri) for _ in range(STEPS)]
            sync_growth(st)
            torch.cuda.synchronize()
        res[rank] = dict(reps=reps, state=st)
    except Exception as e:  # surfaced in the JSON line
        import traceback
        errs.append(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        print(errs[-1], file=sys.stderr, flush=True)
        import os
        os._exit(3)  # the other rank would wait in its next collective forever


threads = [threading.Thread(target=run, args=(r,)) for r in range(WORLD)]
for t in threads:
    t.start()
for t in threads:
    t.join()
if errs:
    print(json.dumps({"ok": False, "errors": errs}))
    sys.exit(0)

faulthandler.cancel_dump_traceback_later()
ref = TrainState(golden_scene(d), TrainConfig(**cfg))
ref_reps = [train_step(ref, views, images, priors, normal_priors=npri) for _ in range(STEPS)]
out = {"ok": True, "loss": [], "param_bad_frac": {}, "owned_disjoint": None}
for s in range(STEPS):
    for r in range(WORLD):
        rb = res[r]["reps"][s]
        out["loss"].append([s, r, rb["rgb"], ref_reps[s].rgb, rb["depth"], ref_reps[s].depth,
                            rb["normal"], ref_reps[s].normal])
        out.setdefault("geo", []).append([s, r, rb.get("geo", 0.0), ref_reps[s].geo,
                                          rb.get("geo_pairs", 0), ref_reps[s].geo_pairs])
owner = res[0]["state"].assignment.flat_owner()
out["owned_disjoint"] = bool(np.array_equal(np.bincount(owner, minlength=WORLD) > 0,
                                            np.ones(WORLD, bool)))
for name in ["emb", "log_scales", "offsets"]:
    want = ref.flat.view(ref.flat.param, name).cpu().numpy()
    got = np.empty_like(want)
    for r in range(WORLD):
        st = res[r]["state"]
        g = st.flat.view(st.flat.param, name).cpu().numpy()
        got[owner == r] = g[owner == r]
    diff = np.abs(got - want)
    bad = diff > 1e-5 * np.maximum(np.abs(got), np.abs(want)) + 1e-7
    out["param_bad_frac"][name] = float(bad.mean())
    # an element whose gradient sits at float32 summation noise (the ranks add
    # the per-view contributions in another order) can take an Adam step of
    # either sign; Adam's update is bounded by lr per step, so any element's
    # divergence is bounded by 2 lr STEPS (lrs at step 0 are the largest)
    lr0 = TrainState(golden_scene(d), TrainConfig(**cfg)).lrs()[name]
    out.setdefault("param_adam_ratio", {})[name] = float(diff.max() / (2 * lr0 * STEPS))
gs_ref = ref.grow_sum_flat.cpu().numpy()
gc_ref = ref.grow_cnt_flat.cpu().numpy()
out["growth_ok"] = all(
    np.array_equal(res[r]["state"].grow_cnt_flat.cpu().numpy(), gc_ref) and
    np.allclose(res[r]["state"].grow_sum_flat.cpu().numpy(), gs_ref, rtol=1e-4, atol=1e-12)
    for r in range(WORLD))
out["growth_nonzero"] = bool(gc_ref.sum() > 0)
for r in range(WORLD):  # the replicated decoder (anchor rows of other owners are stale)
    st = res[r]["state"]
    out[f"dec_checksum_r{r}"] = float(st.flat.view(st.flat.param, "dec/opacity_w1").sum())
out["dec_checksum_ref"] = float(ref.flat.view(ref.flat.param, "dec/opacity_w1").sum())
print(json.dumps(out))
