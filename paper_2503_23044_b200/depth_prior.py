"""Monocular depth-prior alignment and cross-view filtering on the device.

Mirrors voxsplat ``depth_prior.py`` (same names, argument meaning and error
types). The per-point and per-pixel float64 passes run as CUDA kernels behind
the C ABI (``vsx_prior_sample``, ``vsx_apply_scale_shift``,
``vsx_reprojection_error``, ``vsx_enhance_finalize``); the 2x2 normal
equations, the median / MAD refit and the neighbour choice stay on the host
exactly as in the reference (``depth_prior.py:78-214``). Maps are device
tensors: values float64 (H, W), valid bool (H, W).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream
from .errors import DegenerateFit, InsufficientData, InvalidInput
from .geometry import CameraView

MIN_FIT_SAMPLES = 8
MAD_FACTOR = 3.0
VAR_GUARD = 1e-12
Z_EPS = 1e-9
DEFAULT_TAU = 1.0
NEIGHBOR_MIN_DOT = 0.5


def _dev_f64(x) -> torch.Tensor:
    t = x if torch.is_tensor(x) else torch.as_tensor(np.asarray(x, np.float64))
    return t.to(device="cuda", dtype=torch.float64).contiguous()


def _dev_bool(x) -> torch.Tensor:
    t = x if torch.is_tensor(x) else torch.as_tensor(np.asarray(x, bool))
    return t.to(device="cuda", dtype=torch.bool).contiguous()


def _u8(b: torch.Tensor) -> torch.Tensor:
    return b.to(torch.uint8).contiguous()


@dataclass(frozen=True)
class ScaleShiftFit:
    scale: float
    shift: float
    samples: int
    inliers: int


@dataclass
class AlignedDepthMap:
    values: torch.Tensor        # (H, W) float64, metric depth
    valid: torch.Tensor         # (H, W) bool

    def __post_init__(self):
        self.values = _dev_f64(self.values)
        self.valid = _dev_bool(self.valid)
        if self.values.shape != self.valid.shape or self.values.dim() != 2:
            raise InvalidInput("aligned depth map needs matching 2-d value/valid arrays")


@dataclass
class EnhancedDepthMap:
    values: torch.Tensor        # (H, W) float64, zero where invalid
    valid: torch.Tensor         # (H, W) bool
    min_roundtrip: torch.Tensor  # (H, W) float64, inf where never measured
    tau: float


def _solve_scale_shift(d: torch.Tensor, z: torch.Tensor) -> tuple[float, float]:
    """Least-squares (s, b) of z ~ s*d + b from the 2x2 normal equations (:78-82)."""
    sums = torch.stack([(d * d).sum(), d.sum(), (d * z).sum(), z.sum()]).cpu().numpy()
    a = np.array([[sums[0], sums[1]], [sums[1], float(d.numel())]])
    rhs = np.array([sums[2], sums[3]])
    try:
        s, b = np.linalg.solve(a, rhs)
    except np.linalg.LinAlgError as exc:
        raise DegenerateFit("scale/shift normal equations are singular") from exc
    return float(s), float(b)


def _median(x: torch.Tensor) -> float:
    """numpy median semantics (mean of the two middle values for even n)."""
    v, _ = torch.sort(x)
    n = v.numel()
    if n % 2:
        return float(v[n // 2])
    return float((v[n // 2 - 1] + v[n // 2]) / 2)


def fit_scale_shift(depth, view: CameraView, points, valid=None) -> ScaleShiftFit:
    """Fit metric = scale * raw + shift against sparse points seen by `view`
    (``depth_prior.py:85-129``): points projected on the device, raw depth
    sampled bilinearly, one 3-MAD robust refit."""
    depth_t = depth if torch.is_tensor(depth) else torch.as_tensor(np.asarray(depth, np.float64))
    if depth_t.dim() != 2:
        raise InvalidInput("raw depth must be a 2-d array")
    depth_t = _dev_f64(depth_t)
    if valid is None:
        valid_t = torch.isfinite(depth_t) & (depth_t > 0)
    else:
        valid_t = _dev_bool(valid)
    pts = _dev_f64(points).reshape(-1, 3).contiguous()
    n = pts.shape[0]
    raw = torch.empty(n, dtype=torch.float64, device="cuda")
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    ok = torch.empty(n, dtype=torch.uint8, device="cuda")
    valid_u8 = _u8(valid_t)   # bound: a temporary would be freed before the kernel reads it
    call("vsx_prior_sample", ptr(pts), n, view.to_abi(), ptr(depth_t), ptr(valid_u8),
         ptr(raw), ptr(z), ptr(ok), stream())
    projected = int((ok >= 1).sum()) if n else 0
    if projected < MIN_FIT_SAMPLES:
        raise InsufficientData(f"only {projected} projected points, need {MIN_FIT_SAMPLES}")
    sel = ok == 2
    raw, z = raw[sel], z[sel]
    if raw.numel() < MIN_FIT_SAMPLES:
        raise InsufficientData(
            f"only {raw.numel()} samples on valid depth, need {MIN_FIT_SAMPLES}")
    if float(torch.var(raw, unbiased=False)) < VAR_GUARD:
        raise DegenerateFit("raw depth has no variance at the sample points")
    s, b = _solve_scale_shift(raw, z)
    res = s * raw + b - z
    med = _median(res)
    mad = _median(torch.abs(res - med))
    keep = (torch.abs(res - med) <= MAD_FACTOR * mad) if mad >= VAR_GUARD else \
        torch.ones_like(res, dtype=torch.bool)
    inliers = int(keep.sum())
    if inliers >= MIN_FIT_SAMPLES and float(torch.var(raw[keep], unbiased=False)) >= VAR_GUARD:
        s, b = _solve_scale_shift(raw[keep], z[keep])
    else:
        inliers = int(raw.numel())
    if s <= 0:
        raise DegenerateFit(f"non-positive depth scale {s:.3g}")
    return ScaleShiftFit(scale=s, shift=b, samples=int(raw.numel()), inliers=inliers)


def apply_scale_shift(depth, fit: ScaleShiftFit, valid=None) -> AlignedDepthMap:
    """``depth_prior.py:132-140`` on the device."""
    d = _dev_f64(depth)
    out = torch.empty_like(d)
    ov = torch.empty(d.shape, dtype=torch.uint8, device="cuda")
    v = None if valid is None else _u8(_dev_bool(valid))
    call("vsx_apply_scale_shift", ptr(d), ptr(v), d.numel(), float(fit.scale), float(fit.shift),
         ptr(out), ptr(ov), stream())
    return AlignedDepthMap(values=out, valid=ov.bool())


def _check_map(m: AlignedDepthMap, view: CameraView, what: str) -> None:
    if tuple(m.values.shape) != (view.height, view.width):
        raise InvalidInput(f"{what} map shape {tuple(m.values.shape)} != view "
                           f"{(view.height, view.width)}")


def reprojection_error(src: AlignedDepthMap, view_src: CameraView, ref: AlignedDepthMap,
                       view_ref: CameraView, out: torch.Tensor | None = None) -> torch.Tensor:
    """Pixel round-trip error map for every valid source pixel (+inf where the
    chain breaks), ``depth_prior.py:143-187``. With `out`, min-combines into it."""
    _check_map(src, view_src, "source")
    _check_map(ref, view_ref, "reference")
    acc = out is not None
    err = out if acc else torch.empty(src.values.shape, dtype=torch.float64, device="cuda")
    # the uint8 masks are bound to names: two temporaries made inside the
    # argument list would share one recycled block before the kernel runs
    sv, rv = _u8(src.valid), _u8(ref.valid)
    call("vsx_reprojection_error", ptr(src.values), ptr(sv), view_src.to_abi(),
         ptr(ref.values), ptr(rv), view_ref.to_abi(), ptr(err), 1 if acc else 0, stream())
    return err


def select_neighbors(views: list[CameraView], index: int, k: int = 2,
                     min_dot: float = NEIGHBOR_MIN_DOT) -> list[int]:
    """Indices of the k nearest other cameras looking the same general way
    (``depth_prior.py:190-202``; host, O(views))."""
    me = views[index]
    fwd_me = me.r[2]
    scored = []
    for j, v in enumerate(views):
        if j == index:
            continue
        if float(fwd_me @ v.r[2]) < min_dot:
            continue
        scored.append((float(np.linalg.norm(v.center - me.center)), j))
    scored.sort()
    return [j for _, j in scored[:k]]


def enhance(src: AlignedDepthMap, view_src: CameraView,
            neighbors: list[tuple[AlignedDepthMap, CameraView]],
            tau: float = DEFAULT_TAU) -> EnhancedDepthMap:
    """Keep source pixels whose best cross-view round-trip error is <= tau
    (``depth_prior.py:205-214``)."""
    if tau <= 0:
        raise InvalidInput("tau must be positive")
    emin = torch.full(src.values.shape, float("inf"), dtype=torch.float64, device="cuda")
    for ref, view_ref in neighbors:
        reprojection_error(src, view_src, ref, view_ref, out=emin)
    vals = torch.empty_like(src.values)
    ov = torch.empty(src.values.shape, dtype=torch.uint8, device="cuda")
    sv = _u8(src.valid)
    call("vsx_enhance_finalize", ptr(src.values), ptr(sv), ptr(emin), float(tau),
         src.values.numel(), ptr(vals), ptr(ov), stream())
    return EnhancedDepthMap(values=vals, valid=ov.bool(), min_roundtrip=emin, tau=float(tau))


def prepare_depth_priors(views: list[CameraView], raw_depths: list, points,
                         tau: float = DEFAULT_TAU) -> list[EnhancedDepthMap]:
    """Fit, align and cross-view-filter the monocular priors of `views`
    (reference ``trainer.prepare_depth_priors``, ``trainer.py:457-472``, with
    the raw maps passed in instead of read from a dataset)."""
    if len(raw_depths) != len(views):
        raise InvalidInput("one raw depth map per view is required")
    aligned = []
    for v, raw in zip(views, raw_depths):
        fit = fit_scale_shift(raw, v, points)
        aligned.append(apply_scale_shift(raw, fit))
    out = []
    for pos, v in enumerate(views):
        nb = select_neighbors(views, pos)
        out.append(enhance(aligned[pos], v, [(aligned[j], views[j]) for j in nb], tau=tau))
    return out


__all__ = ["ScaleShiftFit", "AlignedDepthMap", "EnhancedDepthMap", "fit_scale_shift",
           "apply_scale_shift", "reprojection_error", "select_neighbors", "enhance",
           "prepare_depth_priors", "MIN_FIT_SAMPLES", "MAD_FACTOR", "VAR_GUARD", "DEFAULT_TAU"]
_ = _lib  # loaded lazily by call()
