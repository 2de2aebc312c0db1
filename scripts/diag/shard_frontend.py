"""Owner-side front end of one rank of an N-rank sharded step, emulated on
one GPU: for 8N views (weak scaling, 8 views per rank) cull + select of the
rank's Eq. 3 shard (every N-th active anchor), decode, projection and the
kept-splat compaction, with the two batched host reads of
CudaShardBackend.forward_shards; timed with CUDA events. ``sort=True`` is the
z-sorted projection the owners used before (the renderer re-sorts anyway).

  python scripts/diag/shard_frontend.py
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2503_23044_b200 import device as D  # noqa: E402
from paper_2503_23044_b200.trainer import TrainConfig, TrainState  # noqa: E402

scene, views, _desc, _ = bench.workload("cfg2")
st = TrainState(scene, TrainConfig(total_steps=100, step2_start=100, step3_start=100,
                                   growth_stop=0))
ds, an = st.dscene, st.anchors
status = torch.zeros(1, dtype=torch.int32, device="cuda")
img = D.decoder_image(st.params.abi(), st.n)
A = ds.count


def group(vs, N, rank, sort):
    own = torch.zeros(A, dtype=torch.bool, device="cuda")
    own[rank::N] = True
    sel = [D.select_async(ds.cull(v) & own.view(torch.uint8)) for v in vs]
    counts = torch.cat([c for _, c in sel]).cpu().tolist()
    launched = []
    for v, (idx, _), c in zip(vs, sel, counts):
        dec = D.decode(st.params.abi(), st.n, idx[:c], ds.centers, an.emb, an.log_scales,
                       an.offsets, v, ds.lod_ref, ds.max_scale, status, keep_cache=True, img=img)
        launched.append(D.project_launch(dec.means, dec.opacity, dec.color, dec.scale, dec.quat,
                                         dec.normal, v, status, sort=sort))
    kept = torch.cat([pl.kept for pl in launched]).cpu().tolist()
    return [D.project_finish(pl, k) for pl, k in zip(launched, kept)]


import time  # noqa: E402

for sort in (False,):
    for N in (1, 8):
        vs = [views[i % len(views)] for i in range(8 * N)]
        for _ in range(2):
            group(vs[:8], N, 0, sort)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h = 0.0
        for g0 in range(0, len(vs), 8):
            t0 = time.perf_counter()
            group(vs[g0:g0 + 8], N, 0, sort)
            h += time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        print(f"  host time in group(): {h * 1e3:.2f} ms ({h * 1e3 / len(vs):.3f} ms per view)")
        print(f"sort={sort} N={N}: owner front end per rank per step ({8 * N} views) {t:.2f} ms",
              flush=True)

# host-side profile of one N=8 group (cProfile, cumulative)
import cProfile  # noqa: E402
import pstats  # noqa: E402
vs = [views[i % len(views)] for i in range(8)]
pr = cProfile.Profile()
pr.enable()
for _ in range(4):
    group(vs, 8, 0, False)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
