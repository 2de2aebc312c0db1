"""The bench's sharded step at world size W on ONE GPU: W threads over
torch's in-process process group (host collectives, so no kernel waits on
another rank's). A crash/consistency smoke test of the multi-GPU bench path
at full size, not a timing: the ranks share one GPU. cfg2: 8 views per rank;
cfg3: 1M anchors, 16 views at 1080p; cfg4: 2M anchors, 8 views at 4K.

  python scripts/threaded_bench_smoke.py [W] [cfg2|cfg3|cfg4]
"""
import sys
import threading
import time
from pathlib import Path

import torch
import torch.distributed as dist
from torch.testing._internal.distributed.multi_threaded_pg import _install_threaded_pg

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2503_23044_b200.dist import CudaShardBackend, sharded_train_step  # noqa: E402
from paper_2503_23044_b200.trainer import TrainConfig, TrainState  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
CONFIG = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
scene, views, desc, _ = bench.workload(CONFIG, W)
print(CONFIG, "anchors", scene.total_voxels, "views", len(views), flush=True)
tgt = bench.teacher_targets(scene, views)
imgs = [t["rgb"] for t in tgt]
priors = [(t["depth"], t["valid"]) for t in tgt]
nprior = [(t["normal"], t["valid"]) for t in tgt]
torch.cuda.init()
torch._C._distributed_c10d._set_thread_isolation_mode(True)
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
out = {}


def run(rank):
    torch.cuda.set_device(0)
    dist.init_process_group("threaded", rank=rank, world_size=W, store=store)
    with torch.cuda.stream(torch.cuda.Stream()):
        cfg = TrainConfig(total_steps=30000, batch_size=len(views), step2_start=0,
                          step3_start=30000, growth_stop=0, normal_weight=0.5, workers=W)
        st = TrainState(scene, cfg)
        be = CudaShardBackend(st, rank, W)
        reps = []
        for _ in range(3):
            t = time.perf_counter()
            r = sharded_train_step(be, views, imgs, priors, nprior)
            torch.cuda.synchronize()
            reps.append((round(time.perf_counter() - t, 3), r["total"], r["rgb"],
                         r.get("imbalance")))
        out[rank] = reps


th = [threading.Thread(target=run, args=(r,)) for r in range(W)]
for t in th:
    t.start()
for t in th:
    t.join()
for r in sorted(out):
    print("rank", r, out[r])
assert len(out) == W
assert all(out[r][-1][1] == out[0][-1][1] for r in out), "ranks disagree on the loss"
print("ok")
