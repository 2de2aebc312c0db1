"""Host-side (Python) cost of the sharded step at world size 1 (cfg2, 8
views): cProfile over a few steps, by internal time. At N ranks an owner
runs the per-view front end and backward tail for 8N views, so per-view
host costs multiply by N.

  python scripts/diag/sharded_host_profile.py
"""
import cProfile
import os
import pstats
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2503_23044_b200.dist import CudaShardBackend, sharded_train_step  # noqa: E402
from paper_2503_23044_b200.trainer import TrainConfig, TrainState  # noqa: E402

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29571", RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl")
scene, views, _desc, _ = bench.workload("cfg2")
tgt = bench.teacher_targets(scene, views)
imgs = [t["rgb"] for t in tgt]
priors = [(t["depth"], t["valid"]) for t in tgt]
nprior = [(t["normal"], t["valid"]) for t in tgt]
cfg = TrainConfig(total_steps=30000, batch_size=len(views), step2_start=0, step3_start=30000,
                  growth_stop=0, normal_weight=0.5)
st = TrainState(scene, cfg)
be = CudaShardBackend(st, 0, 1)
for _ in range(3):
    sharded_train_step(be, views, imgs, priors, nprior)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(3):
    sharded_train_step(be, views, imgs, priors, nprior)
pr.disable()
torch.cuda.synchronize()
print(f"wall per step {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
dist.destroy_process_group()
