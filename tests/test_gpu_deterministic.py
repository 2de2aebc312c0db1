"""Deterministic mode (``TrainConfig.deterministic``).

The reference's sums run in a fixed order, so its steps are bitwise
reproducible (``trainer.py:9-13``). The default B200 path adds per-splat
gradients and loss sums with float atomics, whose order varies run to run.
In deterministic mode the compositor writes per-(splat, tile) gradient rows
and per-(tile, warp) loss partials to fixed slots, reduced in a fixed order
(``vsx_raster_grad_reduce``, ``vsx_reduce_partials``), and the sharded step's
decoder all-reduce becomes an all-gather plus a rank-order sum. These tests
check that two runs are bitwise identical, and that the deterministic sums
equal the atomic ones up to float32 summation order.
"""

from __future__ import annotations

import socket

import numpy as np
import pytest
import torch

from conftest import golden_scene, golden_view

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _inputs(d):
    views = [golden_view(d, f"v{i}", i) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    priors = [(d[f"prior{i}"], d[f"pvalid{i}"]) for i in range(3)]
    rng = np.random.default_rng(5)
    npri = []
    for _ in range(3):
        p = rng.normal(size=(40, 48, 3)).astype(np.float32)
        npri.append((p / np.linalg.norm(p, axis=-1, keepdims=True), rng.uniform(size=(40, 48)) > 0.3))
    return views, images, priors, npri


def _cfg(det: bool) -> dict:
    return dict(total_steps=8, batch_size=3, step2_start=0, step3_start=8, growth_stop=0,
                normal_weight=0.5, deterministic=det)


def _run(d, det: bool, steps: int = 2):
    from paper_2503_23044_b200.trainer import TrainConfig, TrainState, train_step
    views, images, priors, npri = _inputs(d)
    st = TrainState(golden_scene(d), TrainConfig(**_cfg(det)))
    reps = [train_step(st, views, images, priors, normal_priors=npri) for _ in range(steps)]
    torch.cuda.synchronize()
    return st, reps


def test_deterministic_steps_are_bitwise_reproducible(train_small):
    a, ra = _run(train_small, True)
    b, rb = _run(train_small, True)
    assert torch.equal(a.flat.param, b.flat.param)
    assert torch.equal(a.flat.grad, b.flat.grad)
    assert torch.equal(a.grow_sum_flat, b.grow_sum_flat)
    for x, y in zip(ra, rb):
        assert (x.total, x.rgb, x.depth, x.normal) == (y.total, y.rgb, y.depth, y.normal)


def test_deterministic_sums_match_atomic_sums(train_small):
    """One step: the fixed-order gradient equals the atomic one up to the
    float32 summation order. Reordering a sum moves it by up to ~n eps times
    the sum of its summands' magnitudes, which cancellation can make large
    against the result, so the bound is 1e-4 of the element plus 1e-5 of the
    buffer's rms (the per-splat floor of the cfg2 parity tests)."""
    a, ra = _run(train_small, True, steps=1)
    b, rb = _run(train_small, False, steps=1)
    ga, gb = a.flat.grad.double(), b.flat.grad.double()
    rms = float(gb.pow(2).mean().sqrt())
    assert rms > 0
    tol = 1e-4 * gb.abs() + 1e-5 * rms
    worst = float(((ga - gb).abs() / tol).max())
    assert worst <= 1.0, worst
    assert ra[0].rgb == pytest.approx(rb[0].rgb, rel=1e-12)
    assert ra[0].depth == pytest.approx(rb[0].depth, rel=1e-12)
    assert ra[0].normal == pytest.approx(rb[0].normal, rel=1e-12)


def test_deterministic_cfg2_view_gradients():
    """A full 1080p cfg2 view (6.5 M intersections): the deterministic
    per-splat gradients are bitwise reproducible and equal the atomic ones up
    to summation order."""
    import bench
    from paper_2503_23044_b200 import device as D
    from paper_2503_23044_b200._lib import VsxLossDesc
    from paper_2503_23044_b200.trainer import TrainConfig, TrainState
    scene, views, _desc, _ = bench.workload("cfg2")
    v = views[0]
    tgt = bench.teacher_targets(scene, [v])[0]
    st = TrainState(scene, TrainConfig(total_steps=100, step2_start=0, step3_start=100,
                                       growth_stop=0))
    ds = st.dscene
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    act = ds.active(v)
    dec = D.decode(st.params.abi(), st.n, act, ds.centers, st.anchors.emb, st.anchors.log_scales,
                   st.anchors.offsets, v, ds.lod_ref, ds.max_scale, status, keep_cache=False)
    P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, v, status)
    B = D.bin_tiles(P, v.width, v.height)
    H, W = v.height, v.width
    gt = torch.as_tensor(tgt["rgb"]).cuda()
    # a target away from the render so every pixel carries a cotangent
    gt = (gt * 0.9 + 0.05).contiguous()
    pd = torch.as_tensor(tgt["depth"]).cuda() * 1.02
    pv = torch.as_tensor(tgt["valid"]).cuda().to(torch.uint8)

    def run(det: bool):
        sums = torch.zeros(3, dtype=torch.float64, device="cuda")
        counts = torch.zeros(2, dtype=torch.int32, device="cuda")
        loss = VsxLossDesc(gt_rgb=gt.data_ptr(), prior_depth=pd.data_ptr(),
                           prior_depth_valid=pv.data_ptr(), rgb_scale=1.0 / (H * W * 3),
                           depth_weight=1.0, sums=sums.data_ptr(), counts=counts.data_ptr())
        R = D.raster_forward(P, B, v, loss=loss, deterministic=det)
        g = D.raster_backward(P, B, v, R, loss=loss, deterministic=det)
        torch.cuda.synchronize()
        return g.double(), sums.clone()

    g1, s1 = run(True)
    g2, s2 = run(True)
    assert torch.equal(g1, g2) and torch.equal(s1, s2)
    g0, s0 = run(False)
    assert torch.allclose(s1, s0, rtol=1e-12, atol=0)
    rms = g0.pow(2).mean(0).sqrt()               # per gradient field
    tol = 1e-4 * g0.abs() + 1e-5 * rms
    worst = float(((g1 - g0).abs() / tol).max())
    assert worst <= 1.0, worst


def test_deterministic_sharded_world1_matches_train_step(train_small):
    """World size 1 (NCCL): with fixed-order sums the sharded step (C1 self
    exchange, ordered C2) and train_step give the same parameters bit for
    bit."""
    import torch.distributed as dist
    from paper_2503_23044_b200.dist import CudaShardBackend, sharded_train_step
    from paper_2503_23044_b200.trainer import TrainConfig, TrainState, train_step
    d = train_small
    views, images, priors, npri = _inputs(d)
    a = TrainState(golden_scene(d), TrainConfig(**_cfg(True)))
    b = TrainState(golden_scene(d), TrainConfig(**_cfg(True)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", rank=0, world_size=1,
                                init_method=f"tcp://127.0.0.1:{port}")
    try:
        be = CudaShardBackend(b, 0, 1)
        for _ in range(2):
            ra = train_step(a, views, images, priors, normal_priors=npri)
            rb = sharded_train_step(be, views, images, priors, npri)
            # the report divides the same sums in another order: last bit only
            for k in ("rgb", "depth", "normal"):
                assert rb[k] == pytest.approx(getattr(ra, k), rel=1e-15)
    finally:
        if own:
            dist.destroy_process_group()
    torch.cuda.synchronize()
    assert torch.equal(a.flat.param, b.flat.param)


def test_prefetched_inputs_give_the_same_steps(train_small):
    """trainer.StagedInputs (the next step's targets / priors copied to the
    device while the current step runs) is the same computation: with
    fixed-order sums, two steps fed by prefetched inputs equal two steps fed
    by host arrays bit for bit."""
    from paper_2503_23044_b200.trainer import StagedInputs, TrainConfig, TrainState, train_step
    d = train_small
    views, images, priors, npri = _inputs(d)
    a, _ = _run(d, True)
    b = TrainState(golden_scene(d), TrainConfig(**_cfg(True)))
    nxt = StagedInputs(views, images, priors, npri)
    for k in range(2):
        cur = nxt
        if k == 0:
            nxt = StagedInputs(views, images, priors, npri)
        train_step(b, views, cur)
    torch.cuda.synchronize()
    assert torch.equal(a.flat.param, b.flat.param)
