"""Depth-map fusion into a truncated signed distance volume, on the device.

Mirrors voxsplat ``fusion.py`` ``TsdfVolume`` (same constructor, bounds
helper, budget / truncation checks and integrate semantics). The per-voxel
update is the ``vsx_tsdf_integrate`` kernel (float64, reference operation
order); the volume lives in device memory. Marching-cubes mesh extraction
and the KD-tree point-set scores of the reference are not part of this
package.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import call, ptr, stream
from .device import require_cuda
from .errors import InvalidInput, ResourceError
from .geometry import CameraView

DEFAULT_VOXEL_BUDGET = 64_000_000


class TsdfVolume:
    """Dense truncated signed distance volume on a regular grid
    (``fusion.py:40-100``). Voxel (i, j, k) is centred at
    origin + (i, j, k) * voxel_size; tsdf starts at +1, weight at 0."""

    def __init__(self, origin, dims, voxel_size: float, truncation: float,
                 budget: int = DEFAULT_VOXEL_BUDGET):
        require_cuda()
        self.origin = np.asarray(origin, np.float64).reshape(3)
        self.dims = tuple(int(d) for d in dims)
        if len(self.dims) != 3 or min(self.dims) < 2:
            raise InvalidInput(f"volume dims must be three values >= 2, got {dims}")
        if voxel_size <= 0:
            raise InvalidInput("voxel size must be positive")
        if truncation < voxel_size:
            raise InvalidInput(
                f"truncation {truncation:.4g} narrower than one voxel {voxel_size:.4g}")
        total = int(np.prod(self.dims, dtype=np.int64))
        if total > budget:
            raise ResourceError(f"volume of {total} voxels exceeds the budget of {budget}")
        self.voxel_size = float(voxel_size)
        self.truncation = float(truncation)
        self.tsdf = torch.ones(total, dtype=torch.float64, device="cuda")
        self.weight = torch.zeros(total, dtype=torch.float64, device="cuda")

    @classmethod
    def from_bounds(cls, lower, upper, voxel_size: float, truncation: float,
                    budget: int = DEFAULT_VOXEL_BUDGET, auto_coarsen: bool = False):
        """Volume covering an axis-aligned box; with auto_coarsen the voxel
        size (and truncation) doubles until the budget fits (``fusion.py:76-94``)."""
        lower = np.asarray(lower, np.float64).reshape(3)
        upper = np.asarray(upper, np.float64).reshape(3)
        if not (upper > lower).all():
            raise InvalidInput("upper bound must exceed lower bound on every axis")
        vs, tr = float(voxel_size), float(truncation)
        while True:
            dims = np.maximum(np.ceil((upper - lower) / vs).astype(np.int64) + 1, 2)
            total = int(np.prod(dims, dtype=np.int64))
            if total <= budget:
                break
            if not auto_coarsen:
                raise ResourceError(
                    f"volume of {total} voxels exceeds the budget of {budget}; "
                    "enlarge the voxel size or pass auto_coarsen")
            vs *= 2.0
            tr *= 2.0
        return cls(lower, dims, vs, tr, budget=budget)

    @property
    def observed_fraction(self) -> float:
        return float((self.weight > 0).double().mean())

    def integrate(self, depth, valid, view: CameraView) -> int:
        """Fold one depth map into the volume; returns the voxels touched
        (``fusion.py:102-133``)."""
        d = depth if torch.is_tensor(depth) else torch.as_tensor(np.asarray(depth, np.float64))
        m = valid if torch.is_tensor(valid) else torch.as_tensor(np.asarray(valid, bool))
        if tuple(d.shape) != (view.height, view.width) or tuple(m.shape) != tuple(d.shape):
            raise InvalidInput("depth/valid shape must match the view size")
        d = d.to(device="cuda", dtype=torch.float64).contiguous()
        m = m.to(device="cuda", dtype=torch.uint8).contiguous()
        dims = (ctypes.c_int64 * 3)(*self.dims)
        org = (ctypes.c_double * 3)(*[float(x) for x in self.origin])
        touched = torch.zeros(1, dtype=torch.int64, device="cuda")
        call("vsx_tsdf_integrate", ptr(self.tsdf), ptr(self.weight), dims, org, self.voxel_size,
             self.truncation, ptr(d), ptr(m), view.to_abi(), ptr(touched), stream())
        return int(touched.item())

    def grids(self) -> tuple[np.ndarray, np.ndarray]:
        """(tsdf, weight) as host float64 (d0, d1, d2) arrays."""
        return (self.tsdf.cpu().numpy().reshape(self.dims),
                self.weight.cpu().numpy().reshape(self.dims))
