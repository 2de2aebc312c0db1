"""Multi-rank (gloo, CPU) tests of the sharded step's C1/C2 routing.

* exchange round trip: every renderer receives exactly the rows of its views
  from every owner, in source-rank order, and the reverse exchange returns
  each owner the gradients of its own rows;
* end to end: 2 gloo ranks running ``dist.sharded_train_step`` with the
  float64 oracle backend reproduce the single-process oracle train step
  (itself pinned to the reference) for the anchors each rank owns and for the
  replicated decoder.
"""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden_view, load_golden


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            init_method=f"tcp://127.0.0.1:{port}")
    torch.set_num_threads(1)


def _exchange_worker(rank, world, port, out):
    from paper_2503_23044_b200.dist import SplatPayload, exchange_splats, return_grads
    _init(rank, world, port)
    B = 5
    rng = np.random.default_rng(rank)
    payloads = []
    for v in range(B):
        n = int(rng.integers(0, 6)) if (v + rank) % 3 else 0
        gid = torch.tensor([rank * 1000 + v * 100 + i for i in range(n)], dtype=torch.int64)
        rec = gid.double().unsqueeze(-1).repeat(1, 4)
        payloads.append(SplatPayload(rec, gid.double(), gid.double() * 2, gid))
    plan, merged = exchange_splats(payloads, rank, world)
    ok = True
    grads = {}
    for v, (p, seg) in merged.items():
        expect = []
        for q in range(world):
            expect += [q * 1000 + v * 100 + i for i in range(int(plan.counts[q, v]))]
        ok &= p.gid.tolist() == expect and len(seg) == world + 1 and seg[-1] == len(expect)
        grads[v] = p.rec[:, :2] * -1.0
    back = return_grads(plan, grads, torch.zeros((0, 2), dtype=torch.float64))
    for v in range(B):
        ok &= torch.equal(back[v], payloads[v].rec[:, :2] * -1.0)
    torch.save({"ok": bool(ok)}, os.path.join(out, f"r{rank}.pt"))
    dist.destroy_process_group()


def test_exchange_round_trip_two_ranks():
    port = _free_port()
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_exchange_worker, args=(2, port, out), nprocs=2, join=True)
        for r in range(2):
            assert torch.load(os.path.join(out, f"r{r}.pt"))["ok"]


def _c2_worker(rank, world, port, out):
    from paper_2503_23044_b200.dist import _c2_sum
    _init(rank, world, port)
    # values whose float32 sum depends on the order
    base = torch.tensor([1e8, 1.0, -1e8, 3.25, 1e-3], dtype=torch.float32)
    mine = base * (rank + 1) + torch.tensor([0.5, -0.75, 0.125, 2.0, 1e-4]) * rank
    ordered = mine.clone()
    _c2_sum(ordered, None, ordered=True)
    reduced = mine.clone()
    _c2_sum(reduced, None, ordered=False)
    torch.save({"ordered": ordered, "reduced": reduced, "mine": mine},
               os.path.join(out, f"r{rank}.pt"))
    dist.destroy_process_group()


def test_ordered_c2_is_the_rank_order_sum():
    """Deterministic mode's C2: every rank gets the sum accumulated in rank
    order (((g0 + g1) + g2) in float32), whatever the collective's own
    reduction order; the plain all-reduce agrees up to rounding."""
    port = _free_port()
    world = 3
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_c2_worker, args=(world, port, out), nprocs=world, join=True)
        res = [torch.load(os.path.join(out, f"r{r}.pt")) for r in range(world)]
    expect = res[0]["mine"].clone()
    for r in range(1, world):
        expect += res[r]["mine"]
    for r in range(world):
        assert torch.equal(res[r]["ordered"], expect)
        assert torch.allclose(res[r]["reduced"], expect, rtol=1e-6, atol=1e-2)


def _small_state(d):
    import oracle
    K = int(d["lod_count"])
    base = float(d["base_voxel"])
    centers = np.concatenate([d[f"grid{k}"].astype(np.float64) * (base / 2.0 ** k)
                              for k in range(K)])
    levels = np.concatenate([np.full(d[f"grid{k}"].shape[0], k) for k in range(K)])
    n = int(d["n"])
    w = oracle.decoder_init(n, 0, float(np.log(0.125 * base)))
    return oracle.OracleState.create(
        centers, levels, K, float(d["lod_ref"]), int(d["lod_bias"]), base, n, w,
        np.concatenate([d[f"emb{k}"] for k in range(K)]),
        np.log(np.concatenate([d[f"scl{k}"] for k in range(K)])),
        np.concatenate([d[f"off{k}"] for k in range(K)]), total_steps=8, step2_start=0,
        step3_start=8)


def _mixed_priors(d):
    """View 1 without a depth prior, normal priors on views 0 and 2: the terms
    average over the views that carry a prior (trainer.py:296-306)."""
    priors = [(d[f"prior{i}"], d[f"pvalid{i}"]) for i in range(3)]
    priors[1] = None
    rng = np.random.default_rng(5)
    npri = []
    for i in range(3):
        p = rng.normal(size=(40, 48, 3))
        npri.append((p / np.linalg.norm(p, axis=-1, keepdims=True),
                     rng.uniform(size=(40, 48)) > 0.3))
    npri[1] = None
    return priors, npri


def _sharded_worker(rank, world, port, out, case="plain"):
    from oracle.shard import OracleShardBackend
    from paper_2503_23044_b200.dist import sharded_train_step
    from paper_2503_23044_b200.partition import ViewScheduler
    _init(rank, world, port)
    d = load_golden("train_small")
    views = [golden_view(d, f"v{i}", i) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    priors = [(d[f"prior{i}"], d[f"pvalid{i}"]) for i in range(3)]
    npri, wn = None, 0.0
    if case == "mixed":
        priors, npri = _mixed_priors(d)
        wn = 0.5
    st = _small_state(d)
    be = OracleShardBackend(st, rank, world, normal_weight=wn)
    sched = None
    if case == "scheduled":
        # EMA history that moves view 1 to rank 0 and views 0, 2 to rank 1
        sched = ViewScheduler(beta=1.0)
        sched.update(views, [1.0, 5.0, 1.0])
        sched.update = lambda *a, **k: None  # keep the planted assignment
    reps = [sharded_train_step(be, views, images, priors, npri, scheduler=sched)
            for _ in range(2)]
    torch.save({"reps": reps, "owned": be.owned,
                "weights": {k: v.numpy() for k, v in st.weights.items()},
                "emb": st.emb.numpy(), "offsets": st.offsets.numpy(),
                "log_scales": st.log_scales.numpy()}, os.path.join(out, f"r{rank}.pt"))
    dist.destroy_process_group()


@pytest.mark.slow
@pytest.mark.parametrize("case", ["plain", "scheduled", "mixed"])
def test_sharded_step_two_ranks_matches_single_process_oracle(case):
    import oracle
    port = _free_port()
    d = load_golden("train_small")
    views = [golden_view(d, f"v{i}", i) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    priors = [(d[f"prior{i}"], d[f"pvalid{i}"]) for i in range(3)]
    npri, wn = None, 0.0
    if case == "mixed":
        priors, npri = _mixed_priors(d)
        wn = 0.5
    ref = _small_state(d)
    cams = [oracle.Cam.of(v) for v in views]
    ref_reps = [oracle.train_step(ref, cams, images, priors, normal_priors=npri,
                                  normal_weight=wn) for _ in range(2)]
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_sharded_worker, args=(2, port, out, case), nprocs=2, join=True)
        res = [torch.load(os.path.join(out, f"r{r}.pt"), weights_only=False) for r in range(2)]
    for r in res:
        for s in range(2):
            assert r["reps"][s]["rgb"] == pytest.approx(ref_reps[s]["rgb"], rel=1e-10)
            assert r["reps"][s]["depth"] == pytest.approx(ref_reps[s]["depth"], rel=1e-9)
            assert r["reps"][s]["normal"] == pytest.approx(ref_reps[s]["normal"], rel=1e-9,
                                                           abs=1e-15)
            assert r["reps"][s]["total"] == pytest.approx(ref_reps[s]["total"], rel=1e-10)
        for k, w in r["weights"].items():
            np.testing.assert_allclose(w, ref.weights[k].numpy(), rtol=1e-9, atol=1e-13)
        own = r["owned"]
        for name in ("emb", "offsets", "log_scales"):
            np.testing.assert_allclose(r[name][own], getattr(ref, name).numpy()[own],
                                       rtol=1e-9, atol=1e-13)
    assert np.array_equal(res[0]["owned"], ~res[1]["owned"])


def test_sharded_step_refuses_the_ncc_term():
    """With w3 > 0 (step >= step3_start) the sharded step raises instead of
    silently dropping the Eq. 10 term it does not implement."""
    from oracle.shard import OracleShardBackend
    from paper_2503_23044_b200.dist import sharded_train_step
    from paper_2503_23044_b200.errors import InvalidInput
    port = _free_port()
    dist.init_process_group("gloo", rank=0, world_size=1,
                            init_method=f"tcp://127.0.0.1:{port}")
    try:
        d = load_golden("train_small")
        views = [golden_view(d, f"v{i}", i) for i in range(3)]
        images = [d[f"img{i}"] for i in range(3)]
        st = _small_state(d)
        st.step3_start, st.step = 0, 1
        with pytest.raises(InvalidInput):
            sharded_train_step(OracleShardBackend(st, 0, 1), views, images)
    finally:
        dist.destroy_process_group()
