"""f4 .vsnap state IO: byte-compatible container, reference checkpoint
resume (snapshot.py, trainer.py:491-522)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, golden_scene, golden_view, load_golden


@pytest.fixture(scope="module")
def ck():
    return load_golden("checkpoint")


def test_reader_matches_reference_records(ck):
    from paper_2503_23044_b200.snapshot import read_snapshot
    data = read_snapshot(GOLDEN / "checkpoint.vsnap")
    got = {f"{tag}:{n}": a for tag, rec in data.items() for n, a in rec.items()}
    ref = {k: v for k, v in ck.items() if ":" in k}
    assert list(got) == list(ref)
    for k, a in ref.items():
        assert got[k].dtype == a.dtype and got[k].shape == a.shape, k
        np.testing.assert_array_equal(got[k], a, err_msg=k)


def test_writer_reproduces_reference_bytes(tmp_path):
    from paper_2503_23044_b200.snapshot import read_snapshot, write_snapshot
    src = GOLDEN / "checkpoint.vsnap"
    data = read_snapshot(src)
    out = write_snapshot(tmp_path / "copy.vsnap", list(data.items()))
    assert out.read_bytes() == src.read_bytes()


def test_reader_rejects_corruption(tmp_path):
    from paper_2503_23044_b200.errors import IoError
    from paper_2503_23044_b200.snapshot import read_snapshot
    blob = (GOLDEN / "checkpoint.vsnap").read_bytes()
    for name, bad in (("magic", b"XXXXX\0" + blob[6:]), ("trunc", blob[:-7]),
                      ("trail", blob + b"\0"), ("version", blob[:6] + b"\x02" + blob[7:])):
        p = tmp_path / f"{name}.vsnap"
        p.write_bytes(bad)
        with pytest.raises(IoError):
            read_snapshot(p)


def test_scene_records_round_trip():
    from paper_2503_23044_b200.snapshot import read_snapshot, scene_from_records, \
        scene_to_records
    data = read_snapshot(GOLDEN / "checkpoint.vsnap")
    scene = scene_from_records(data["SCNE"])
    assert scene.lod_count == 2 and scene.offsets_per_voxel == 3 and "TRN1" in data
    again = scene_to_records(scene)
    assert list(again) == list(data["SCNE"])
    for k, a in data["SCNE"].items():
        np.testing.assert_array_equal(again[k], a, err_msg=k)


@pytest.mark.gpu
def test_resume_reference_checkpoint_matches_reference(ck, train_small):
    from paper_2503_23044_b200.trainer import TrainConfig, load_checkpoint, train_step
    from gpu_util import rel_close
    d = train_small
    views = [golden_view(d, f"v{i}", i) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    cfg = TrainConfig(total_steps=8, batch_size=3, step2_start=8, step3_start=8, growth_stop=0)
    state = load_checkpoint(GOLDEN / "checkpoint.vsnap", cfg)
    assert state.step == 2
    rep = train_step(state, views, images)
    np.testing.assert_allclose([rep.total, rep.rgb, rep.step], ck["resume_loss"], rtol=2e-4)
    for name in [k[len("resume_post_"):] for k in ck if k.startswith("resume_post_")
                 and "_lv" not in k]:
        got = state.flat.view(state.flat.param, f"dec/{name}").detach().cpu().numpy()
        ok, worst, nbad = rel_close(got, ck[f"resume_post_{name}"], 1e-3, 1e-6)
        assert nbad / got.size <= 5e-3, f"{name}: {nbad}/{got.size}, worst {worst:.3g}"
    for key, flat in (("embeddings", "emb"), ("log_scales", "log_scales"),
                      ("offsets", "offsets")):
        ref = np.concatenate([ck[f"resume_post_lv{k}_{key}"].reshape(-1) for k in range(2)])
        got = state.flat.view(state.flat.param, flat).detach().cpu().numpy().reshape(-1)
        ok, worst, nbad = rel_close(got, ref, 1e-3, 1e-6)
        assert nbad / got.size <= 5e-3, f"{key}: {nbad}/{got.size}, worst {worst:.3g}"


@pytest.mark.gpu
def test_save_load_round_trip(tmp_path, train_small):
    import torch
    from paper_2503_23044_b200.trainer import (TrainConfig, TrainState, load_checkpoint,
                                               save_checkpoint, train_step)
    d = train_small
    views = [golden_view(d, f"v{i}", i) for i in range(3)]
    images = [d[f"img{i}"] for i in range(3)]
    cfg = TrainConfig(total_steps=8, batch_size=3, step2_start=8, step3_start=8, growth_stop=0)
    state = TrainState(golden_scene(d), cfg)
    train_step(state, views, images)
    path = save_checkpoint(tmp_path / "s.vsnap", state)
    back = load_checkpoint(path, cfg)
    assert back.step == state.step
    for buf in ("param", "m", "v"):
        a, b = getattr(state.flat, buf), getattr(back.flat, buf)
        torch.testing.assert_close(a, b, rtol=0, atol=0)
    assert back.rng.bit_generator.state == state.rng.bit_generator.state
    r1 = train_step(state, views, images)
    r2 = train_step(back, views, images)
    assert r1.total == pytest.approx(r2.total, rel=1e-6)
