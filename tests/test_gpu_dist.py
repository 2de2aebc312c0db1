"""The sharded (C1/C2) CUDA path on one GPU: a world-size-1 NCCL group runs the
same exchange code paths (all-to-all, merge + lexsort((gid, z)), reverse
all-to-all, decoder all-reduce) and must reproduce ``train_step``."""

from __future__ import annotations

import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from conftest import golden_scene, golden_view

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    yield
    dist.destroy_process_group()


def test_sort_z_gid_is_lexsort():
    from paper_2503_23044_b200 import device as D
    rng = np.random.default_rng(0)
    z = np.round(rng.uniform(1, 2, 50000), 3)           # many exact ties
    gid = rng.permutation(50000).astype(np.int64)
    order = D.sort_z_gid(torch.as_tensor(z).cuda(), torch.as_tensor(gid).cuda()).cpu().numpy()
    np.testing.assert_array_equal(order, np.lexsort((gid, z)))


def test_c1_rows_pack_keys_gather_roundtrip():
    """The CUDA C1 row path: rows packed by vsx_pack_splat_rows, keys read
    back through a row map (rows of one view from several sources), and the
    records / radii gathered in (z, gid) order equal torch indexing."""
    from ctypes import c_void_p
    from paper_2503_23044_b200 import device as D
    from paper_2503_23044_b200._lib import call, ptr, stream
    from paper_2503_23044_b200.dist import ROW_BYTES, SplatPayload, _pack_rows
    g = torch.Generator(device="cuda").manual_seed(5)
    parts = []
    for n in (1000, 0, 2500, 777):
        rec = torch.randn((n, 16), device="cuda", generator=g)
        z = torch.rand(n, device="cuda", generator=g, dtype=torch.float64).round(decimals=2) + 1
        rad = torch.rand(n, device="cuda", generator=g, dtype=torch.float64) * 30
        gid = torch.randperm(10 ** 6, device="cuda", generator=g)[:n]
        parts.append(SplatPayload(rec, z, rad, gid))
    total = sum(p.count for p in parts)
    buf = _pack_rows(parts, total, "cuda")
    assert buf.shape == (total, ROW_BYTES)
    cat = SplatPayload.cat(parts, parts[0])
    # the "view" takes part 3 then part 0 (two source blocks)
    offs = np.cumsum([0] + [p.count for p in parts])
    rowmap = torch.cat([torch.arange(offs[3], offs[4]), torch.arange(offs[0], offs[1])]).int().cuda()
    n = int(rowmap.numel())
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    gid = torch.empty(n, dtype=torch.int64, device="cuda")
    call("vsx_splat_rows_keys", c_void_p(buf.data_ptr()), ptr(rowmap), n, ptr(z), ptr(gid), stream())
    rl = rowmap.long()
    assert torch.equal(z, cat.z[rl]) and torch.equal(gid, cat.gid[rl])
    order = D.sort_z_gid(z, gid, int32=True)
    rs = torch.empty((n, 16), device="cuda")
    rr = torch.empty(n, dtype=torch.float64, device="cuda")
    call("vsx_gather_splat_rows", c_void_p(buf.data_ptr()), ptr(rowmap), ptr(order), n, ptr(rs),
         ptr(rr), stream())
    src = rl[order.long()]
    assert torch.equal(rs, cat.rec[src]) and torch.equal(rr, cat.radius[src])


def test_sharded_step_world1_matches_train_step(nccl_world1, train_small):
    """World size 1 (NCCL self-exchange) against train_step: losses to float
    rounding of the report and, with fixed-order sums
    (TrainConfig.deterministic), parameters bit for bit."""
    from paper_2503_23044_b200.dist import CudaShardBackend, sharded_train_step
    from paper_2503_23044_b200.trainer import TrainConfig, TrainState, train_step
    d = train_small
    views = [golden_view(d, f"v{i}", i) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    priors = [(d[f"prior{i}"], d[f"pvalid{i}"]) for i in range(3)]
    cfg = dict(total_steps=8, batch_size=3, step2_start=0, step3_start=8, growth_stop=0,
               deterministic=True)
    a = TrainState(golden_scene(d), TrainConfig(**cfg))
    b = TrainState(golden_scene(d), TrainConfig(**cfg))
    be = CudaShardBackend(b, 0, 1)
    for _ in range(2):
        ra = train_step(a, views, images, priors)
        rb = sharded_train_step(be, views, images, priors)
        assert rb["rgb"] == pytest.approx(ra.rgb, rel=1e-15)
        assert rb["depth"] == pytest.approx(ra.depth, rel=1e-15)
    torch.cuda.synchronize()
    assert torch.equal(a.flat.param, b.flat.param)


@pytest.mark.parametrize("world,nv,geo", [(2, 3, False), (4, 3, False), (4, 2, False),
                                         (3, 2, False), (2, 3, True), (4, 2, True)])
def test_sharded_step_threaded_ranks_match_train_step(world, nv, geo):
    """World size 2 and 4 on one GPU: threads of one process joined by
    torch's in-process process group (host-side collectives, no cross-rank
    kernel waits). Losses on every rank and the owner-merged anchor
    parameters must match the single-process train_step; the replicated
    decoder too. At world 4 with 3 views one rank renders nothing. One view
    has no depth prior and one no normal prior (per-term normalisation over
    the views that carry one), and the growth accumulators summed over the
    ranks equal train_step's. With fewer views than ranks (4 ranks / 2
    views, 3 ranks / 2 views) every view is split into tile-row bands
    rendered on different ranks: the per-view valid-pixel counts are summed
    over the bands before the backward, and owners add each splat's band
    gradients. With the Eq. 10 NCC term (w3 > 0 from step 1) every rank
    receives all renders and evaluates the term with the same RNG draws:
    the term's value and pair count match train_step's on every rank."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    p = subprocess.run([sys.executable, str(here / "dist_threaded_worker.py"), str(world),
                        str(nv)] + (["geo"] if geo else []),
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["ok"], "\n".join(out.get("errors", []))[-3000:]
    for s, r, rgb, ref_rgb, dep, ref_dep, nrm, ref_nrm in out["loss"]:
        assert rgb == pytest.approx(ref_rgb, rel=1e-6), (s, r)
        assert dep == pytest.approx(ref_dep, rel=1e-5), (s, r)
        assert nrm == pytest.approx(ref_nrm, rel=1e-5), (s, r)
    for s, r, g, ref_g, gp, ref_gp in out["geo"]:
        assert gp == ref_gp, (s, r)
        assert g == pytest.approx(ref_g, rel=1e-5, abs=1e-9), (s, r)
    if geo:
        assert any(g > 0 for _, _, g, _, _, _ in out["geo"])
    # growth pressure accumulated by the owners, summed over ranks = train_step's
    assert out["growth_nonzero"] and out["growth_ok"]
    # element-wise: within 1e-5 rel, except near-zero-gradient Adam sign flips
    # (float32 summation order across ranks), which are bounded by Adam's
    # 2 lr per step and must stay rare
    for name, frac in out["param_bad_frac"].items():
        assert frac < 1e-2, (name, frac)
        assert out["param_adam_ratio"][name] <= 1.0, (name, out["param_adam_ratio"][name])
    for r in range(world):
        assert out[f"dec_checksum_r{r}"] == pytest.approx(out["dec_checksum_ref"], rel=1e-5)
