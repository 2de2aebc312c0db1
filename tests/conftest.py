"""Shared test configuration: markers, fixture loaders, golden-case builders."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / round-end)")
    config.addinivalue_line("markers", "slow: multi-second CPU oracle runs")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as f:
        return {k: f[k] for k in f.files}


def golden_view(d: dict, prefix: str, view_id: int = 0):
    from paper_2503_23044_b200.geometry import CameraView
    fx, fy, cx, cy = d[f"{prefix}_intr"]
    w, h = d[f"{prefix}_size"]
    return CameraView(view_id, int(w), int(h), float(fx), float(fy), float(cx), float(cy),
                      d[f"{prefix}_r"], d[f"{prefix}_t"])


def golden_scene(d: dict):
    """Rebuild a SceneModel from stored reference arrays (no RNG involved)."""
    from paper_2503_23044_b200.scene import SceneLevel, SceneModel
    K = int(d["lod_count"])
    base = float(d["base_voxel"])
    levels = []
    for k in range(K):
        v = d[f"grid{k}"].shape[0]
        levels.append(SceneLevel(k, base / 2.0 ** k, d[f"grid{k}"], d[f"emb{k}"],
                                 d[f"scl{k}"], d[f"off{k}"], np.zeros(v, np.int32)))
    return SceneModel(base, K, int(d["n"]), levels, lod_ref_distance=float(d["lod_ref"]),
                      lod_bias=int(d["lod_bias"]))


@pytest.fixture(scope="session")
def scene_small():
    return load_golden("scene_small")


@pytest.fixture(scope="session")
def raster_leaf():
    return load_golden("raster_leaf")


@pytest.fixture(scope="session")
def train_small():
    return load_golden("train_small")


@pytest.fixture(scope="session")
def cfg1_golden():
    path = GOLDEN / "cfg1.npz"
    if not path.exists():
        pytest.skip("cfg1 golden fixture not generated")
    return load_golden("cfg1")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
