"""One rank of an N-rank sharded step, owner side, emulated on one GPU:
CudaShardBackend's forward_shards over 8N views (groups of 8) on the rank's
Eq. 3 anchor shard (every N-th anchor), then backward_shard of every view
with zero 2D gradients. Reports host wall time and GPU time; at N ranks
this owner work runs beside the rank's compositing of its 8 views
(~15 ms of GPU time per step at cfg2).

  python scripts/diag/shard_rank_emu.py
"""
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2503_23044_b200 import device as D  # noqa: E402
from paper_2503_23044_b200.dist import CudaShardBackend  # noqa: E402
from paper_2503_23044_b200.trainer import TrainConfig, TrainState  # noqa: E402

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29572", RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl")
scene, views, _desc, _ = bench.workload("cfg2")
cfg = TrainConfig(total_steps=30000, batch_size=len(views), step2_start=0, step3_start=30000,
                  growth_stop=0, normal_weight=0.5)
st = TrainState(scene, cfg)
be = CudaShardBackend(st, 0, 1)
_ = be.owned   # builds the cache key


def owner_step(N):
    vs = [views[i % len(views)] for i in range(8 * N)]
    be.begin_step(vs)
    own = torch.zeros(st.dscene.count, dtype=torch.uint8, device="cuda")
    own[0::N] = 1
    be._owned = own   # the cached Eq. 3 mask of rank 0 of N (key unchanged)
    pay = {}
    for g0 in range(0, len(vs), 8):
        gen = be.forward_shards(list(range(g0, min(g0 + 8, len(vs)))), vs)
        try:
            while True:
                next(gen)
        except StopIteration as e:
            pay.update(e.value)
    for v in range(len(vs)):
        grads = torch.zeros((pay[v].count, D.GRAD_F32), dtype=torch.float32, device="cuda")
        be.backward_shard(v, vs[v], grads)


for N in (1, 2, 4, 8):
    owner_step(N)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    owner_step(N)
    h = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    print(f"N={N}: owner work per rank per step ({8 * N} views): host {h * 1e3:.1f} ms, "
          f"GPU span {e0.elapsed_time(e1):.1f} ms", flush=True)
if os.environ.get("EMU_PROFILE") == "1":
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    owner_step(8)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("cumtime").print_stats(40)
dist.destroy_process_group()
