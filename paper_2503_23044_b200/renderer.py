"""Rasterizer API of ``voxsplat/renderer.py`` over the B200 kernels K3-K7.

``project_splats`` (K3 + stable radix sort), ``bin_splats`` (K4),
``rasterize_view`` (K5) return device tensors; the reference's numpy
bookkeeping (radius, zkey, gid, owner, per-tile counts) is materialised
lazily. Gradients flow through torch autograd Functions whose backward
passes are the hand-written kernels (``vsx_raster_bwd`` K6,
``vsx_project_bwd`` K7), so ``rasterize_backward`` keeps the reference's
contract (``renderer.py:347-367``).
"""

from __future__ import annotations

import copy
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as D
from .decoder import DecoderParams, GaussianBatch, decode_active, quat_to_rotmat_t
from .errors import ContractViolation, InvalidInput, TransferError
from .geometry import CameraView
from .partition import PATCH, PatchRect, WorkerAssignment

Z_NEAR = 0.01
ALPHA_CLAMP = 0.99
EARLY_STOP_T = 1e-4
ALPHA_VALID_MIN = 1e-4
DENOM_GUARD = 1e-6
LOWPASS = 0.3
BYTES_PER_GAUSSIAN = 17 * 8     # reference accounting unit (renderer.py:45)
SPLAT_RECORD_BYTES = 64         # what the B200 exchange actually moves per splat
ALL_TASKS = frozenset({"rgb", "depth", "normal", "alpha"})


class ProjectedSplats:
    """Screen-space splats of one view, sorted by (camera z, gaussian id)."""

    def __init__(self, P: D.Projected, batch: GaussianBatch, feat: torch.Tensor | None,
                 view: CameraView):
        self._P = P
        self._batch = batch
        self.feat = feat            # (G', 13) autograd carrier when graph-connected
        self.view = view
        self.leaves = batch.leaves
        self._bins: D.Bins | None = None

    @property
    def count(self) -> int:
        return self._P.count

    mean2d = property(lambda self: self._P.mean2d)
    conic = property(lambda self: self._P.conic)
    color = property(lambda self: self._P.color)
    opacity = property(lambda self: self._P.opacity)
    normal_cam = property(lambda self: self._P.normal_cam)
    plane_d = property(lambda self: self._P.plane_d)

    @property
    def radius(self) -> np.ndarray:
        return self._P.radius.cpu().numpy()

    @property
    def zkey(self) -> np.ndarray:
        return self._P.zkey.cpu().numpy().view(np.float64)

    @property
    def src(self) -> np.ndarray:
        return self._P.src.cpu().numpy().astype(np.int64)

    @property
    def gid(self) -> np.ndarray:
        return self._batch.gid[self.src]

    @property
    def owner(self) -> np.ndarray:
        return self._batch.owner[self.src]

    def bins(self) -> D.Bins:
        if self._bins is None:
            self._bins = D.bin_tiles(self._P, self.view.width, self.view.height)
        return self._bins

    def assert_sorted(self) -> None:
        if self.count < 2:
            return
        z = self.zkey
        gid = self.gid
        dz = np.diff(z)
        if np.any(dz < 0) or np.any(np.diff(gid)[dz == 0] <= 0):
            raise ContractViolation("splats are not sorted by (z, gid)")


@dataclass
class TransferStats:
    gaussians: int
    bytes_moved: int
    per_worker_bytes: np.ndarray


@dataclass
class RenderTargets:
    rgb: torch.Tensor
    depth: torch.Tensor
    normal: torch.Tensor
    alpha: torch.Tensor
    valid: torch.Tensor
    raw_normal: torch.Tensor
    aux: D.Raster | None = None

    def to_numpy(self) -> dict[str, np.ndarray]:
        out = {k: getattr(self, k).detach().cpu().numpy().astype(np.float64)
               for k in ("rgb", "depth", "normal", "alpha")}
        out["valid"] = self.valid.cpu().numpy().astype(bool)
        return out


@dataclass
class RenderStats:
    gaussians: int = 0
    tile_splat_counts: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    elapsed_seconds: float = 0.0
    transfer: TransferStats | None = None


# ------------------------------------------------------------------ autograd bridges

class _ProjectFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, view, box, means, opac, color, scale, quat, normal):
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        P = D.project(means, opac, color, scale, quat, normal, view, status)
        D.check_status(status, "project_splats")
        box.append(P)
        ctx.view, ctx.P = view, P
        ctx.save_for_backward(means, scale, quat, normal)
        return torch.zeros((P.count, D.GRAD_F32), dtype=torch.float32, device="cuda")

    @staticmethod
    def backward(ctx, gfeat):
        means, scale, quat, normal = ctx.saved_tensors
        g = D.project_backward(means, scale.detach().float().contiguous(),
                               quat.detach().float().contiguous(),
                               normal.detach().float().contiguous(), ctx.P,
                               gfeat.float().contiguous(), ctx.view)
        return (None, None, g["means"].to(means.dtype), g["opacities"], g["colors"],
                g["scales"], g["quats"], g["normals"])


class _RasterFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, feat, P, B, view, box):
        R = D.raster_forward(P, B, view)
        box.append(R)
        ctx.P, ctx.B, ctx.view, ctx.R = P, B, view, R
        ctx.mark_non_differentiable(R.valid)
        return R.rgb, R.alpha, R.depth, R.normal, R.raw_normal, R.valid

    @staticmethod
    def backward(ctx, g_rgb, g_alpha, g_depth, g_normal, g_raw, _g_valid):
        c = lambda t: None if t is None else t.float().contiguous()  # noqa: E731
        grad = D.raster_backward(ctx.P, ctx.B, ctx.view, ctx.R, c(g_rgb), c(g_alpha), c(g_depth),
                                 c(g_normal), c(g_raw))
        return grad, None, None, None, None


# ------------------------------------------------------------------ API

def make_leaf_gaussians(means, opacities, colors, scales, quats, normals=None,
                        requires_grad: bool = False) -> GaussianBatch:
    """Raw gaussian leaves on the device (``renderer.py:110-141``)."""
    D.require_cuda()
    f32 = lambda a, shape: torch.as_tensor(np.asarray(a, np.float32)).reshape(shape).cuda()  # noqa: E731
    leaves = {"means": torch.as_tensor(np.asarray(means, np.float64)).reshape(-1, 3).cuda(),
              "opacities": f32(opacities, (-1,)), "colors": f32(colors, (-1, 3)),
              "scales": f32(scales, (-1, 3)), "quats": f32(quats, (-1, 4))}
    if requires_grad:
        for t in leaves.values():
            t.requires_grad_(True)
    q = leaves["quats"] / torch.linalg.norm(leaves["quats"], dim=-1, keepdim=True).clamp_min(1e-12)
    if normals is None:
        rot = quat_to_rotmat_t(q)
        axis = torch.argmin(leaves["scales"], dim=-1)
        nrm = torch.take_along_dim(rot, axis[:, None, None].expand(-1, 3, 1), -1).squeeze(-1)
    else:
        nrm = f32(normals, (-1, 3))
    return GaussianBatch(leaves["means"], leaves["opacities"], leaves["colors"], leaves["scales"],
                         q, nrm, leaves=leaves if requires_grad else None)


def project_splats(batch: GaussianBatch, view: CameraView) -> ProjectedSplats:
    """EWA projection and (z, gid) sort (``renderer.py:144-204``)."""
    D.require_cuda()
    ins = [batch.means, batch.opacities, batch.colors, batch.scales, batch.quats, batch.normals]
    box: list = []
    grad_on = torch.is_grad_enabled() and any(t.requires_grad for t in ins)
    if grad_on:
        feat = _ProjectFn.apply(view, box, *[t.contiguous() for t in ins])
        P = box[0]
    else:
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        P = D.project(*[t.detach().contiguous() for t in ins], view, status)
        D.check_status(status, "project_splats")
        feat = None
    return ProjectedSplats(P, batch, feat, view)


def bin_splats(splats: ProjectedSplats, width: int, height: int) -> list[np.ndarray]:
    """Per-tile ascending splat index lists (``renderer.py:207-226``)."""
    if (width, height) != (splats.view.width, splats.view.height):
        B = D.bin_tiles(splats._P, width, height)
    else:
        B = splats.bins()
    off = B.tile_offsets.cpu().numpy().astype(np.int64)
    lst = B.tile_list.cpu().numpy().astype(np.int64)
    return [lst[off[t]:off[t + 1]] for t in range(B.tiles_x * B.tiles_y)]


def splats_for_rect(splats: ProjectedSplats, x0: int, y0: int, w: int, h: int) -> np.ndarray:
    """Splats whose 3-sigma box meets a pixel rect (``renderer.py:229-239``)."""
    m = splats.mean2d.cpu().numpy()
    r = splats.radius
    u, v = m[:, 0], m[:, 1]
    hit = (u + r >= x0) & (u - r < x0 + w) & (v + r >= y0) & (v - r < y0 + h)
    return np.flatnonzero(hit)


def rasterize_view(splats: ProjectedSplats, view: CameraView,
                   tasks: frozenset[str] = ALL_TASKS) -> tuple[RenderTargets, np.ndarray]:
    """Blend every tile of a view (``renderer.py:390-449``); returns per-tile counts."""
    B = splats.bins()
    box: list = []
    if splats.feat is not None and torch.is_grad_enabled():
        rgb, alpha, depth, normal, raw, valid = _RasterFn.apply(splats.feat, splats._P, B, view, box)
        R = box[0]
    else:
        R = D.raster_forward(splats._P, B, view)
        rgb, alpha, depth, normal, raw, valid = R.rgb, R.alpha, R.depth, R.normal, R.raw_normal, R.valid
    valid_b = valid.bool() if "depth" in tasks else (alpha.detach() >= ALPHA_VALID_MIN)
    counts = torch.diff(B.tile_offsets.long()).cpu().numpy()
    return RenderTargets(rgb, depth, normal, alpha, valid_b, raw, aux=R), counts


def rasterize_patch(patch: PatchRect, splats: ProjectedSplats, view: CameraView,
                    tasks: frozenset[str] = ALL_TASKS, indices: np.ndarray | None = None) -> dict:
    """Blend exactly the splats ``indices`` (default: ``splats_for_rect`` of
    the rectangle) over every pixel of one pixel rectangle
    (``renderer.py:304-344``); returns (h, w[, c]) tensors plus 'valid'.

    Runs the K5 kernel on a virtual (w x h) image whose origin is the
    rectangle's corner: the selected records are gathered in their (z, gid)
    order with the mean shifted by (-x0, -y0), the principal point likewise,
    and every 16x16 sub-tile lists all of them (the reference blends the
    whole overlap set at every pixel of the patch, no per-tile cut). A
    tile-aligned 16x16 patch with its bin list equals rasterize_view's tile.
    Differentiable through the projected splats when they carry a graph.
    """
    splats.assert_sorted()
    if indices is None:
        indices = splats_for_rect(splats, patch.x0, patch.y0, patch.width, patch.height)
    indices = np.asarray(indices, np.int64)
    if indices.size > 1 and np.any(np.diff(indices) <= 0):
        raise ContractViolation("patch splat indices must be ascending")
    w, h = int(patch.width), int(patch.height)
    if w <= 0 or h <= 0:
        raise InvalidInput("patch must have a positive size")
    # the virtual view: same pose and focal lengths, origin at the corner (its
    # principal point may lie outside the rectangle, so no re-validation)
    sub_view = copy.copy(view)
    sub_view.width, sub_view.height = w, h
    sub_view.cx, sub_view.cy = view.cx - patch.x0, view.cy - patch.y0
    n = int(indices.size)
    if n == 0:
        z = torch.zeros((h, w), dtype=torch.float32, device="cuda")
        out = {"alpha": z.clone(), "valid": torch.zeros((h, w), dtype=torch.bool, device="cuda")}
        for k, c in (("rgb", 3), ("depth", 0), ("normal", 3)):
            if k in tasks:
                out[k] = torch.zeros((h, w, c) if c else (h, w), device="cuda")
        return out
    idx = torch.as_tensor(indices, device="cuda")
    P = splats._P
    rec = P.rec[idx].clone()
    rec.view(torch.float64)[:, 0:2] -= torch.tensor([float(patch.x0), float(patch.y0)],
                                                    dtype=torch.float64, device="cuda")
    sub = D.Projected(rec, P.radius[idx], P.zkey[idx], P.src[idx], n)
    txn, tyn = (w + 15) // 16, (h + 15) // 16
    T = txn * tyn
    offs = (torch.arange(T + 1, device="cuda", dtype=torch.int64) * n).to(torch.int32)
    lst = torch.arange(n, device="cuda", dtype=torch.int32).repeat(T)
    B = D.Bins(offs, lst, txn, tyn)
    box: list = []
    if splats.feat is not None and torch.is_grad_enabled():
        rgb, alpha, depth, normal, raw, valid = _RasterFn.apply(splats.feat[idx], sub, B, sub_view,
                                                                box)
    else:
        R = D.raster_forward(sub, B, sub_view)
        rgb, alpha, depth, normal, valid = R.rgb, R.alpha, R.depth, R.normal, R.valid
    valid_b = valid.bool() if "depth" in tasks else (alpha.detach() >= ALPHA_VALID_MIN)
    out = {"valid": valid_b, "alpha": alpha}
    for k, t in (("rgb", rgb), ("depth", depth), ("normal", normal)):
        if k in tasks:
            out[k] = t
    return out


def rasterize_backward(splats: ProjectedSplats, outputs: dict, upstream: dict) -> dict:
    """Gradients of render outputs w.r.t. the 3D leaves (``renderer.py:347-367``)."""
    if splats.leaves is None:
        raise InvalidInput("splats were not projected from leaf tensors")
    outs, cots = [], []
    for k, t in outputs.items():
        if k in upstream and upstream[k] is not None and t.is_floating_point() and t.requires_grad:
            outs.append(t)
            u = upstream[k]
            u = u if torch.is_tensor(u) else torch.as_tensor(np.asarray(u))
            cots.append(u.to(device=t.device, dtype=t.dtype).reshape(t.shape))
    if not outs:
        raise InvalidInput("no upstream gradients supplied")
    names = list(splats.leaves)
    grads = torch.autograd.grad(outs, [splats.leaves[n] for n in names], grad_outputs=cots,
                                retain_graph=True, allow_unused=True)
    return {n: (g if g is not None else torch.zeros_like(splats.leaves[n]))
            for n, g in zip(names, grads)}


def transfer_gaussians(view: CameraView, scene, assignment: WorkerAssignment,
                       params: DecoderParams, renderer_workers: frozenset[int] = frozenset({0}),
                       state=None, keep_graph: bool = False):
    """Decode the view's active set and account cross-worker bytes (``renderer.py:452-477``)."""
    batch = decode_active(params, scene, view, state=state, keep_graph=keep_graph)
    per_worker = np.zeros(assignment.num_workers, dtype=np.int64)
    if batch.count:
        owners = batch.owner
        counts = np.bincount(owners, minlength=assignment.num_workers)
        for w in renderer_workers:
            if w >= assignment.num_workers:
                raise InvalidInput(f"renderer worker {w} out of range")
            foreign = batch.count - int(counts[w])
            per_worker[w] = foreign * BYTES_PER_GAUSSIAN
            if foreign and assignment.unreachable:
                bad = set(np.unique(owners).tolist()) & (set(assignment.unreachable) - {w})
                if bad:
                    raise TransferError(f"owner worker(s) {sorted(bad)} unreachable")
    return batch, TransferStats(batch.count, int(per_worker.sum()), per_worker)


def render_view(view: CameraView, scene, assignment: WorkerAssignment, params: DecoderParams,
                tasks: frozenset[str] = ALL_TASKS,
                renderer_workers: frozenset[int] = frozenset({0}), state=None,
                keep_graph: bool = False):
    """Decode + project + rasterize one view (``renderer.py:480-493``)."""
    t0 = time.perf_counter()
    batch, tstats = transfer_gaussians(view, scene, assignment, params, renderer_workers,
                                       state, keep_graph)
    splats = project_splats(batch, view)
    targets, counts = rasterize_view(splats, view, tasks)
    torch.cuda.synchronize()
    return targets, RenderStats(batch.count, counts, time.perf_counter() - t0, tstats)


def render_gaussians(view: CameraView, means, opacities, colors, scales, quats, normals=None,
                     tasks: frozenset[str] = ALL_TASKS, requires_grad: bool = False):
    batch = make_leaf_gaussians(means, opacities, colors, scales, quats, normals, requires_grad)
    splats = project_splats(batch, view)
    targets, _ = rasterize_view(splats, view, tasks)
    return targets, splats
