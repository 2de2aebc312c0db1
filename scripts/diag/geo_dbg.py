"""Debug: sharded NCC path at world 1 (NCCL) vs train_step, step 1."""
import socket, sys
import numpy as np, torch
import torch.distributed as dist
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import golden_scene, golden_view, load_golden
from paper_2503_23044_b200 import dist as D
from paper_2503_23044_b200.trainer import TrainConfig, TrainState, train_step
d = load_golden("train_small")
views = [golden_view(d, f"v{i}", i) for i in range(3)]
images = [d[f"img{i}"] for i in range(3)]
cfg = dict(total_steps=8, batch_size=3, step2_start=8, step3_start=0, growth_stop=0)
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
dist.init_process_group("nccl", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
import paper_2503_23044_b200.losses as L
orig_geo = L.geo_loss_cotangents
def geo_spy(tg, views, rng, **k):
    for i, t in enumerate(tg):
        print("  tg", i, float(t.alpha.sum()), int(t.valid.bool().sum()), float(t.normal.abs().sum()),
              float(t.depth.sum()), float(t.rgb.sum()), file=sys.stderr)
    print("  rng state", rng.bit_generator.state["state"]["state"] % 1000003, file=sys.stderr)
    return orig_geo(tg, views, rng, **k)
L.geo_loss_cotangents = geo_spy
orig = D._exchange_renders_and_geo
def wrapped(*a, **k):
    r = orig(*a, **k)
    print("geo called", r[0], r[1].pairs_used, r[1].patches_used, file=sys.stderr)
    return r
D._exchange_renders_and_geo = wrapped
a = TrainState(golden_scene(d), TrainConfig(**cfg)); b = TrainState(golden_scene(d), TrainConfig(**cfg))
be = D.CudaShardBackend(b, 0, 1)
for k in range(2):
    print("schedule", be.schedule(), file=sys.stderr)
    ra = train_step(a, views, images)
    rb = D.sharded_train_step(be, views, images)
    print(k, "ref", ra.geo, ra.geo_pairs, "sharded", rb.get("geo"), rb.get("geo_pairs"), file=sys.stderr)
dist.destroy_process_group()
