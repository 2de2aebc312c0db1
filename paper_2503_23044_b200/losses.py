"""Photometric and depth losses (``voxsplat/losses.py:43-95``) on the device.

``bl_rgb_loss`` / ``e_depth_loss`` keep the reference signatures and return
differentiable scalars (autograd Functions whose forward and backward are
the ``vsx_l1_loss`` / ``vsx_depth_loss`` kernels). The trainer calls the
kernels directly and fuses the cotangent images into the raster backward.
"""

from __future__ import annotations

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
