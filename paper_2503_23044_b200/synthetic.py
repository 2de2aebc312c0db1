"""Synthetic workloads named by BASELINE.json (host-side scene builders).

* :func:`cfg1_scene` — the CPU-runnable parity config:
  120k points on a thin slab, 10,198 anchors x 10 gaussians, 4 views 128^2.
* :func:`city_scene` — the aerial city block of cfg2/cfg3 (ground plane +
  a grid of box buildings), sized by anchor count, with oblique 1080p views.
"""

from __future__ import annotations

import numpy as np

from .geometry import CameraView, look_at
from .scene import SparsePoints, build_hierarchy


def cfg1_scene(seed: int = 0):
    """Scene, views and GT images of cfg1 (same RNG stream as the survey recipe)."""
    rng = np.random.default_rng(seed)
    pts = np.stack([rng.uniform(-1, 1, 120000), rng.uniform(-1, 1, 120000),
                    rng.uniform(-0.005, 0.005, 120000)], -1)
    scene = build_hierarchy(SparsePoints(pts), base_voxel_size=0.02, lod_count=1,
                            offsets_per_voxel=10, seed=0)
    f = 64.0 / np.tan(np.radians(30.0))
    views = []
    for i in range(4):
        eye = np.array([0.3 * np.cos(np.pi * i / 2), 0.3 * np.sin(np.pi * i / 2), 2.2])
        r, t = look_at(eye, np.zeros(3), up=(0.0, 1.0, 0.0))
        views.append(CameraView(i, 128, 128, f, f, 63.5, 63.5, r, t))
    scene.set_lod_reference(views)
    images = [rng.uniform(0, 1, (128, 128, 3)) for _ in range(4)]
    return scene, views, images
