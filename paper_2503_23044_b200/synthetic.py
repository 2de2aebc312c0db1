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


def _box_faces(center, size):
    """Four walls + roof of an axis-aligned building (bottom face is never seen)."""
    c = np.asarray(center, np.float64)
    s = np.asarray(size, np.float64) / 2.0
    faces = []
    for axis in (0, 1):
        for sign in (-1.0, 1.0):
            other = 1 - axis
            faces.append((c + np.eye(3)[axis] * sign * s[axis], axis, other, s[other], s[2]))
    faces.append((c + np.array([0.0, 0.0, s[2]]), 2, 0, s[0], s[1]))
    return faces


def city_points(blocks: int = 12, extent: float = 30.0, n_points: int = 1_500_000,
                seed: int = 0) -> np.ndarray:
    """Surface samples of a ground plane plus a grid of box buildings.

    Area-uniform sampling over the ground and every visible building face
    (the recipe of the reference's synthetic primitives, ``synthetic.py:30-91``
    and ``:265-277``), so anchors spread over all surfaces.
    """
    rng = np.random.default_rng(seed)
    pitch = 2 * extent / blocks
    quads = [(np.zeros(3), 2, 0, extent, extent)]          # ground, normal +z
    for i in range(blocks):
        for j in range(blocks):
            cx = -extent + (i + 0.5) * pitch
            cy = -extent + (j + 0.5) * pitch
            w, d = rng.uniform(0.35, 0.7, 2) * pitch
            h = rng.uniform(0.3, 1.6) * pitch
            quads += _box_faces((cx, cy, h / 2.0), (w, d, h))
    areas = np.array([4 * q[3] * q[4] for q in quads])
    pick = rng.choice(len(quads), size=n_points, p=areas / areas.sum())
    uv = rng.uniform(-1.0, 1.0, size=(n_points, 2))
    centers = np.stack([q[0] for q in quads])
    u_axis = np.array([q[2] for q in quads])
    v_axis = 3 - np.array([q[1] for q in quads]) - u_axis
    half = np.array([[q[3], q[4]] for q in quads])
    pts = centers[pick].copy()
    rows = np.arange(n_points)
    pts[rows, u_axis[pick]] += uv[:, 0] * half[pick, 0]
    pts[rows, v_axis[pick]] += uv[:, 1] * half[pick, 1]
    return pts


def city_views(count: int = 8, width: int = 1920, height: int = 1080, extent: float = 30.0,
               radius: float = 34.0, height_m: float = 26.0, fov_deg: float = 60.0,
               first_id: int = 0) -> list[CameraView]:
    """Oblique aerial orbit looking at the block centre (``synthetic.py:340-353`` pattern)."""
    views = []
    for i in range(count):
        ang = 2 * np.pi * (i + 0.5) / count
        eye = np.array([radius * np.cos(ang), radius * np.sin(ang), height_m])
        tgt = np.array([0.15 * extent * np.cos(ang + 1.0), 0.15 * extent * np.sin(ang + 1.0), 0.0])
        r, t = look_at(eye, tgt)
        f = 0.5 * width / np.tan(np.radians(fov_deg) / 2.0)
        views.append(CameraView(first_id + i, width, height, f, f, (width - 1) / 2.0,
                                (height - 1) / 2.0, r, t))
    return views


def city_scene(target_anchors: int = 200_000, lod_count: int = 3, n: int = 10,
               n_views: int = 8, width: int = 1920, height: int = 1080, seed: int = 0,
               base_voxel_size: float | None = None):
    """cfg2/cfg3: aerial city block sized to ~target_anchors anchors (all levels)."""
    pts = city_points(n_points=max(600_000, int(7.5 * target_anchors)), seed=seed)
    views = city_views(n_views, width, height)
    if base_voxel_size is None:
        base_voxel_size = _fit_voxel(pts, target_anchors, lod_count)
    scene = build_hierarchy(SparsePoints(pts), base_voxel_size, lod_count,
                            offsets_per_voxel=n, seed=seed, views=views)
    return scene, views


def _fit_voxel(pts: np.ndarray, target: int, lod_count: int) -> float:
    from .scene import quantize

    def total(delta: float) -> int:
        return sum(np.unique(quantize(pts, delta / 2.0 ** k), axis=0).shape[0]
                   for k in range(lod_count))

    lo, hi = 0.05, 8.0
    for _ in range(18):
        mid = np.sqrt(lo * hi)
        if total(mid) > target:
            lo = mid
        else:
            hi = mid
    return float(hi)
