"""TEST INFRASTRUCTURE ONLY — float64 CPU restatement of the f1 prior path.

Restates voxsplat ``depth_prior.py`` (scale/shift fit, alignment, cross-view
round trip, enhance) so the device kernels in ``csrc/depth_prior.cu`` have a
checker. Only tests/ may import it. Pinned against the reference's own
outputs in ``tests/golden/depth_prior.npz`` (``oracle/make_golden.py``).
"""

from __future__ import annotations

import numpy as np

MIN_SAMPLES = 8          # depth_prior.py:23
MAD_K = 3.0              # :24
VAR_EPS = 1e-12          # :25
Z_MIN = 1e-9             # :26


class Cam:
    """Pinhole camera: world->camera (r, t), intrinsics, size."""

    def __init__(self, r, t, fx, fy, cx, cy, width, height):
        self.r = np.asarray(r, np.float64).reshape(3, 3)
        self.t = np.asarray(t, np.float64).reshape(3)
        self.fx, self.fy, self.cx, self.cy = float(fx), float(fy), float(cx), float(cy)
        self.width, self.height = int(width), int(height)

    @property
    def center(self):
        return -self.r.T @ self.t

    def to_cam(self, p):
        return np.asarray(p, np.float64) @ self.r.T + self.t

    def to_world(self, c):
        return (np.asarray(c, np.float64) - self.t) @ self.r

    def project(self, c):
        """(u, v, in_front) of camera-frame points (safe divide where behind)."""
        front = c[:, 2] > Z_MIN
        z = np.where(front, c[:, 2], 1.0)
        return self.fx * c[:, 0] / z + self.cx, self.fy * c[:, 1] / z + self.cy, front

    def inside(self, u, v):
        return (u >= 0) & (u <= self.width - 1) & (v >= 0) & (v <= self.height - 1)


def sample_bilinear(vals, ok, u, v):
    """Bilinear sample needing all four texels valid (depth_prior.py:62-74)."""
    h, w = vals.shape
    iu = np.clip(np.floor(u), 0, w - 2).astype(np.int64)
    iv = np.clip(np.floor(v), 0, h - 2).astype(np.int64)
    a, b = u - iu, v - iv
    good = ok[iv, iu] & ok[iv, iu + 1] & ok[iv + 1, iu] & ok[iv + 1, iu + 1]
    s = (vals[iv, iu] * (1 - a) * (1 - b) + vals[iv, iu + 1] * a * (1 - b)
         + vals[iv + 1, iu] * (1 - a) * b + vals[iv + 1, iu + 1] * a * b)
    return s, good


def _ls(d, z):
    """Normal equations of z ~ s d + b (depth_prior.py:78-82)."""
    m = np.array([[d @ d, d.sum()], [d.sum(), float(len(d))]])
    return tuple(float(x) for x in np.linalg.solve(m, np.array([d @ z, z.sum()])))


def fit(depth, cam: Cam, points, valid=None):
    """(scale, shift, samples, inliers) as depth_prior.py:85-129; raises
    ValueError where the reference raises InsufficientData / DegenerateFit."""
    depth = np.asarray(depth, np.float64)
    if valid is None:
        valid = np.isfinite(depth) & (depth > 0)
    c = cam.to_cam(np.asarray(points, np.float64).reshape(-1, 3))
    u, v, front = cam.project(c)
    keep = front & cam.inside(u, v)
    if keep.sum() < MIN_SAMPLES:
        raise ValueError("insufficient projected points")
    raw, good = sample_bilinear(depth, valid, u[keep], v[keep])
    raw, z = raw[good], c[keep, 2][good]
    if len(raw) < MIN_SAMPLES:
        raise ValueError("insufficient valid samples")
    if np.var(raw) < VAR_EPS:
        raise ValueError("degenerate")
    s, b = _ls(raw, z)
    r = s * raw + b - z
    med = np.median(r)
    mad = np.median(np.abs(r - med))
    inl = np.abs(r - med) <= MAD_K * mad if mad >= VAR_EPS else np.ones(len(r), bool)
    n_in = int(inl.sum())
    if n_in >= MIN_SAMPLES and np.var(raw[inl]) >= VAR_EPS:
        s, b = _ls(raw[inl], z[inl])
    else:
        n_in = len(raw)
    if s <= 0:
        raise ValueError("non-positive scale")
    return s, b, len(raw), n_in


def align(depth, scale, shift, valid=None):
    """depth_prior.py:132-140 -> (values, valid)."""
    depth = np.asarray(depth, np.float64)
    if valid is None:
        valid = np.isfinite(depth) & (depth > 0)
    m = scale * depth + shift
    ok = np.asarray(valid, bool) & np.isfinite(m) & (m > 0)
    return np.where(ok, m, 0.0), ok


def round_trip(src_vals, src_ok, cs: Cam, ref_vals, ref_ok, cr: Cam):
    """Round-trip pixel error src -> ref -> src (depth_prior.py:143-187)."""
    out = np.full(src_vals.shape, np.inf)
    iv, iu = np.nonzero(src_ok)
    if iu.size == 0:
        return out
    z = src_vals[iv, iu]
    pc = np.stack([(iu - cs.cx) / cs.fx * z, (iv - cs.cy) / cs.fy * z, z], -1)
    in_ref = cr.to_cam(cs.to_world(pc))
    ur, vr, good = cr.project(in_ref)
    good &= cr.inside(ur, vr)
    if not good.any():
        return out
    zs, sgood = sample_bilinear(ref_vals, ref_ok, np.where(good, ur, 0.0), np.where(good, vr, 0.0))
    good &= sgood & (zs > 0)
    back = np.stack([(ur - cr.cx) / cr.fx * zs, (vr - cr.cy) / cr.fy * zs, zs], -1)
    in_src = cs.to_cam(cr.to_world(back))
    u2, v2, front = cs.project(in_src)
    good &= front
    e = np.hypot(u2 - iu, v2 - iv)
    out[iv[good], iu[good]] = e[good]
    return out


def neighbours(cams, index, k=2, min_dot=0.5):
    """depth_prior.py:190-202."""
    me = cams[index]
    cand = sorted((float(np.linalg.norm(c.center - me.center)), j) for j, c in enumerate(cams)
                  if j != index and float(me.r[2] @ c.r[2]) >= min_dot)
    return [j for _, j in cand[:k]]


def enhance(src_vals, src_ok, cs: Cam, refs, tau):
    """depth_prior.py:205-214 -> (values, valid, min_roundtrip)."""
    emin = np.full(src_vals.shape, np.inf)
    for vals, ok, cr in refs:
        emin = np.minimum(emin, round_trip(src_vals, src_ok, cs, vals, ok, cr))
    keep = src_ok & (emin <= tau)
    return np.where(keep, src_vals, 0.0), keep, emin
