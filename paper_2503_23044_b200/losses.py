"""Photometric and depth losses (``voxsplat/losses.py:43-95``) on the device.

``bl_rgb_loss`` / ``e_depth_loss`` keep the reference signatures and return
differentiable scalars (autograd Functions whose forward and backward are
the ``vsx_l1_loss`` / ``vsx_depth_loss`` kernels). The trainer calls the
kernels directly and fuses the cotangent images into the raster backward.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._lib import call, ptr, stream
from .device import require_cuda
from .errors import InvalidInput


def _as_dev(x, like: torch.Tensor) -> torch.Tensor:
    t = x if torch.is_tensor(x) else torch.as_tensor(np.asarray(x))
    return t.to(device=like.device, dtype=torch.float32).contiguous()


class _L1Fn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, rendered, target, scale):
        acc = torch.zeros(1, dtype=torch.float64, device=rendered.device)
        grad = torch.empty_like(rendered)
        call("vsx_l1_loss", ptr(rendered), ptr(target), rendered.numel(), float(scale), ptr(acc),
             ptr(grad), stream())
        ctx.save_for_backward(grad)
        return (acc * scale).to(torch.float32).reshape(())

    @staticmethod
    def backward(ctx, g):
        (grad,) = ctx.saved_tensors
        return grad * g, None, None


def bl_rgb_loss(rendered: list, reference: list) -> torch.Tensor:
    """Mean over views of mean |I_hat - I|."""
    if len(rendered) != len(reference) or not rendered:
        raise InvalidInput("batch lists must be equal length and non-empty")
    require_cuda()
    terms = []
    for r, g in zip(rendered, reference):
        g = _as_dev(g, r)
        if tuple(r.shape) != tuple(g.shape):
            raise InvalidInput(f"image shape mismatch {tuple(r.shape)} vs {tuple(g.shape)}")
        r32 = r if r.dtype == torch.float32 else r.float()
        terms.append(_L1Fn.apply(r32.contiguous(), g, 1.0 / (r.numel() * len(rendered))))
    return torch.stack(terms).sum()


def loss_bl_rgb(rendered: list, reference: list):
    leaves = [torch.as_tensor(np.asarray(r, np.float32)).cuda().requires_grad_(True)
              for r in rendered]
    val = bl_rgb_loss(leaves, reference)
    grads = torch.autograd.grad(val, leaves)
    return float(val), [g.cpu().numpy() for g in grads]


class _DepthFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, depth, valid, prior, pvalid):
        sums = torch.zeros(1, dtype=torch.float64, device=depth.device)
        cnt = torch.zeros(1, dtype=torch.int32, device=depth.device)
        call("vsx_depth_loss", ptr(depth), ptr(valid), ptr(prior), ptr(pvalid), depth.numel(),
             ptr(sums), ptr(cnt), ptr(None), ptr(None), stream())
        n = int(cnt.item())
        ctx.n = n
        ctx.save_for_backward(depth, valid, prior, pvalid)
        val = (sums / n).float().reshape(()) if n else torch.zeros((), device=depth.device)
        return val, torch.tensor(n)

    @staticmethod
    def backward(ctx, g, _gn):
        depth, valid, prior, pvalid = ctx.saved_tensors
        if ctx.n == 0:
            return torch.zeros_like(depth), None, None, None
        scale = (g.float() / ctx.n).reshape(1).contiguous()
        grad = torch.empty_like(depth)
        call("vsx_depth_loss", ptr(depth), ptr(valid), ptr(prior), ptr(pvalid), depth.numel(),
             ptr(None), ptr(None), ptr(scale), ptr(grad), stream())
        return grad, None, None, None


def e_depth_loss(rendered_depth: list, rendered_valid: list, prior_depth: list,
                 prior_valid: list) -> tuple[torch.Tensor, int]:
    """Masked depth L1 over prior-kept & render-valid pixels; (loss, supervised px)."""
    if not rendered_depth or len({len(rendered_depth), len(rendered_valid), len(prior_depth),
                                  len(prior_valid)}) != 1:
        raise InvalidInput("depth loss needs aligned non-empty batch lists")
    terms, total = [], 0
    for d, dv, p, pv in zip(rendered_depth, rendered_valid, prior_depth, prior_valid):
        d32 = d if d.dtype == torch.float32 else d.float()
        val, n = _DepthFn.apply(d32.contiguous(), _as_dev(dv, d).to(torch.uint8),
                                _as_dev(p, d), _as_dev(pv, d).to(torch.uint8))
        terms.append(val)
        total += int(n)
    return torch.stack(terms).mean(), total


# ------------------------------------------------------------------ Eq. 10 NCC

GRAY_WEIGHTS = (0.299, 0.587, 0.114)
NCC_STD_GUARD = 1e-6
PLANE_D_GUARD = 1e-6
GEO_ALPHA_MIN = 0.9


def pair_views(views: list) -> list[tuple[int, int]]:
    """Greedy proximity chain over camera centres, then consecutive
    (reference, source) pairs (losses.py:155-168; host)."""
    if len(views) < 2:
        return []
    centres = np.stack([v.center for v in views])
    rest = list(range(1, len(views)))
    chain = [0]
    while rest:
        d = [np.linalg.norm(centres[j] - centres[chain[-1]]) for j in rest]
        chain.append(rest.pop(int(np.argmin(d))))
    return [(chain[i], chain[i + 1]) for i in range(0, len(chain) - 1, 2)]


def stratified_centers(cand_u: np.ndarray, cand_v: np.ndarray, width: int, height: int,
                       count: int, rng: np.random.Generator) -> np.ndarray:
    """Up to `count` candidate indices spread over a ceil(sqrt(count))^2 cell
    grid (losses.py:177-196): per cell (ascending id) one rng.permutation of
    its candidates in index order, then round-robin pops from the back. Same
    RNG draws as the reference, vectorised except for the <= count picks."""
    cells = int(np.ceil(np.sqrt(count)))
    cw = max(width / cells, 1.0)
    ch = max(height / cells, 1.0)
    cell_id = (cand_v / ch).astype(np.int64) * cells + (cand_u / cw).astype(np.int64)
    order = np.argsort(cell_id, kind="stable")
    ids = cell_id[order]
    if ids.size == 0:
        return np.zeros(0, np.int64)
    starts = np.flatnonzero(np.r_[True, ids[1:] != ids[:-1]])
    ends = np.r_[starts[1:], ids.size]
    queues = [rng.permutation(order[s:e]) for s, e in zip(starts, ends)]
    picked: list[int] = []
    r = 0
    while len(picked) < count and any(q.size > r for q in queues):
        for q in queues:
            if q.size > r and len(picked) < count:
                picked.append(int(q[q.size - 1 - r]))
        r += 1
    return np.asarray(picked, dtype=np.int64)


@dataclass
class GeoLossStats:
    pairs_used: int = 0
    patches_used: int = 0
    patches_rejected: int = 0


def _ncc_geom(vs, vr):
    from ._lib import VsxNccGeom
    r_rel = vr.r @ vs.r.T
    t_rel = vr.t - r_rel @ vs.t
    g = VsxNccGeom()
    g.r_rel[:] = [float(x) for x in r_rel.reshape(-1)]
    g.t_rel[:] = [float(x) for x in t_rel]
    g.src_fx, g.src_fy, g.src_cx, g.src_cy = float(vs.fx), float(vs.fy), float(vs.cx), float(vs.cy)
    g.ref_fx, g.ref_fy, g.ref_cx, g.ref_cy = float(vr.fx), float(vr.fy), float(vr.cx), float(vr.cy)
    return g


def geo_loss_cotangents(targets: list, views: list, rng: np.random.Generator,
                        patch_count: int = 64, half: int = 3, upstream: float = 1.0):
    """Eq. 10 value and its cotangents (losses.py:199-287) on the device.

    Returns (loss, stats, cot) with loss a float64 device scalar (mean over
    used pairs of the mean 1 - NCC of the pair's patches), and cot a dict
    view index -> (g_rgb, g_normal, g_depth) float32 images holding
    upstream * d loss / d(rendered rgb, normal, depth) of each source view.
    Reference colours are a stop-gradient branch (no cotangent).
    """
    stats = GeoLossStats()
    dev = "cuda"
    pairs_used = torch.zeros(1, dtype=torch.int32, device=dev)
    records = []
    N = (2 * half + 1) ** 2
    for ref_i, src_i in pair_views(views):
        src, ref = targets[src_i], targets[ref_i]
        vs, vr = views[src_i], views[ref_i]
        h, w = vs.height, vs.width
        cand = (src.alpha.detach() > GEO_ALPHA_MIN) & src.valid.bool() & \
            (torch.linalg.vector_norm(src.normal.detach(), dim=-1) > 0.5)
        cand[:half, :] = False
        cand[h - half:, :] = False
        cand[:, :half] = False
        cand[:, w - half:] = False
        vv, uu = (x.cpu().numpy() for x in torch.nonzero(cand, as_tuple=True))
        if uu.size == 0:
            continue
        pick = stratified_centers(uu.astype(np.float64), vv.astype(np.float64), w, h,
                                  patch_count, rng)
        cen = torch.as_tensor(np.stack([uu[pick], vv[pick]], -1).astype(np.int32)).to(dev)
        P = int(pick.size)
        rec = {"src": src_i, "centers": cen, "P": P,
               "term": torch.empty(P, dtype=torch.float64, device=dev),
               "status": torch.empty(P, dtype=torch.uint8, device=dev),
               "g_patch": torch.empty((P, N), dtype=torch.float64, device=dev),
               "g_n": torch.empty((P, 3), dtype=torch.float64, device=dev),
               "g_dep": torch.empty(P, dtype=torch.float64, device=dev),
               "sum": torch.zeros(1, dtype=torch.float64, device=dev),
               "used": torch.zeros(1, dtype=torch.int32, device=dev)}
        # operands bound to names: a temporary made inside the call's argument
        # list would be freed (and its block reused by the next temporary)
        # before the kernel reads it
        srgb = src.rgb.detach().float().contiguous()
        snrm = src.normal.detach().float().contiguous()
        sdep = src.depth.detach().float().contiguous()
        rrgb = ref.rgb.detach().float().contiguous()
        call("vsx_ncc_patches", ptr(srgb), ptr(snrm), ptr(sdep), w, h,
             ptr(rrgb), vr.width, vr.height, _ncc_geom(vs, vr),
             ptr(cen), P, half, ptr(rec["term"]), ptr(rec["status"]), ptr(rec["g_patch"]),
             ptr(rec["g_n"]), ptr(rec["g_dep"]), ptr(rec["sum"]), ptr(rec["used"]),
             ptr(pairs_used), stream())
        records.append(rec)
    cot = {}
    if not records:
        return torch.zeros((), dtype=torch.float64, device=dev), stats, cot
    used = torch.cat([r["used"] for r in records])
    sums = torch.cat([r["sum"] for r in records])
    per_pair = torch.where(used > 0, sums / used.clamp_min(1).double(), torch.zeros_like(sums))
    n_pairs = pairs_used.double().clamp_min(1.0)
    loss = per_pair.sum() / n_pairs[0]
    stats.pairs_used = int(pairs_used.item())
    stats.patches_used = int(used.sum())
    stats.patches_rejected = int(sum(int((r["status"] != 2).sum()) for r in records))
    for r in records:
        vs = views[r["src"]]
        if r["src"] not in cot:
            cot[r["src"]] = (torch.zeros((vs.height, vs.width, 3), dtype=torch.float32, device=dev),
                             torch.zeros((vs.height, vs.width, 3), dtype=torch.float32, device=dev),
                             torch.zeros((vs.height, vs.width), dtype=torch.float32, device=dev))
        g_rgb, g_nrm, g_dep = cot[r["src"]]
        call("vsx_ncc_scatter", ptr(r["centers"]), r["P"], half, vs.width, ptr(r["status"]),
             ptr(r["g_patch"]), ptr(r["g_n"]), ptr(r["g_dep"]), ptr(r["used"]), ptr(pairs_used),
             float(upstream), ptr(g_rgb), ptr(g_nrm), ptr(g_dep), stream())
    return loss, stats, cot


class _GeoFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, value, cots, *tensors):
        ctx.cots = cots
        return value.clone()

    @staticmethod
    def backward(ctx, g):
        return (None, None) + tuple(c * g.to(c.dtype) for c in ctx.cots)


def bl_geo_loss(targets: list, views: list, rng: np.random.Generator, patch_count: int = 64,
                half: int = 3) -> tuple[torch.Tensor, GeoLossStats]:
    """Multi-view patch NCC loss (losses.py:199-287): a differentiable scalar
    w.r.t. the source views' rendered rgb / normal / depth tensors."""
    require_cuda()
    loss, stats, cot = geo_loss_cotangents(targets, views, rng, patch_count, half, 1.0)
    ins, cts = [], []
    for vi, (g_rgb, g_nrm, g_dep) in cot.items():
        t = targets[vi]
        for x, c in ((t.rgb, g_rgb), (t.normal, g_nrm), (t.depth, g_dep)):
            ins.append(x)
            cts.append(c.to(x.dtype))
    return _GeoFn.apply(loss, cts, *ins), stats
