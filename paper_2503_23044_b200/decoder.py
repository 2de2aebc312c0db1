"""Shared gaussian decoder on the device (API of ``voxsplat/decoder.py``).

Weights are float32 CUDA tensors with the reference names and layouts
(``decoder.py:39-98``). ``decode_active`` runs culling (K1) and the decode
kernel (K2) and returns a :class:`GaussianBatch` of device tensors in the
canonical (level, voxel, slot) order; with ``keep_graph=True`` the batch is
differentiable through ``vsx_decode_bwd`` (K8) via a torch autograd Function.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import VsxDecoder, VsxDecoderGrads, call, ptr, stream
from .device import (Decoded, check_status, decode as _decode, device_scene_for,
                     require_cuda, workspace)
from .errors import InvalidInput, ProtocolError, StateError
from .geometry import CameraView

HIDDEN = 64
IN_DIM = 36
HEADS = ("opacity", "color", "cov")
HEAD_WIDTH = {"opacity": 1, "color": 3, "cov": 7}
MIN_SCALE = 1e-6


class DecoderParams:
    """The twelve decoder tensors (float32, CUDA) plus offsets-per-voxel ``n``."""

    def __init__(self, n: int, tensors: dict[str, torch.Tensor] | None = None):
        self.n = int(n)
        self.tensors = tensors if tensors is not None else {}

    @staticmethod
    def param_names(n: int) -> list[str]:
        return [f"{h}_{p}" for h in HEADS for p in ("w1", "b1", "w2", "b2")]

    @staticmethod
    def shapes(n: int) -> dict[str, tuple]:
        out = {}
        for h in HEADS:
            w = HEAD_WIDTH[h] * n
            out.update({f"{h}_w1": (IN_DIM, HIDDEN), f"{h}_b1": (HIDDEN,),
                        f"{h}_w2": (HIDDEN, w), f"{h}_b2": (w,)})
        return out

    @staticmethod
    def init_arrays(n: int, seed: int = 0, scale_bias: float | None = None) -> dict:
        """Host float64 draws in the reference order (decoder.py:54-78)."""
        if n < 1:
            raise InvalidInput("offsets per voxel must be >= 1")
        rng = np.random.default_rng(seed)
        arrays = {}
        for h in HEADS:
            w = HEAD_WIDTH[h] * n
            lim1, lim2 = 1.0 / np.sqrt(IN_DIM), 1.0 / np.sqrt(HIDDEN)
            arrays[f"{h}_w1"] = rng.uniform(-lim1, lim1, (IN_DIM, HIDDEN))
            arrays[f"{h}_b1"] = np.zeros(HIDDEN)
            arrays[f"{h}_w2"] = rng.uniform(-lim2, lim2, (HIDDEN, w))
            arrays[f"{h}_b2"] = np.zeros(w)
        if scale_bias is not None:
            arrays["cov_b2"].reshape(n, 7)[:, 0:3] = float(scale_bias)
        return arrays

    @classmethod
    def init(cls, n: int, seed: int = 0, scale_bias: float | None = None) -> "DecoderParams":
        return cls.from_arrays(n, cls.init_arrays(n, seed, scale_bias))

    @classmethod
    def from_arrays(cls, n: int, arrays: dict) -> "DecoderParams":
        require_cuda()
        t = {}
        for name in cls.param_names(n):
            if name not in arrays:
                raise InvalidInput(f"decoder arrays missing {name}")
            t[name] = torch.as_tensor(np.asarray(arrays[name], np.float32)).cuda().contiguous()
        return cls(n, t)

    def to_arrays(self) -> dict[str, np.ndarray]:
        return {k: v.detach().double().cpu().numpy() for k, v in self.tensors.items()}

    def clone(self) -> "DecoderParams":
        return DecoderParams(self.n, {k: v.detach().clone() for k, v in self.tensors.items()})

    def requires_grad_(self, flag: bool = True) -> "DecoderParams":
        for v in self.tensors.values():
            v.requires_grad_(flag)
        return self

    def abi(self) -> VsxDecoder:
        d = VsxDecoder()
        for h, head in enumerate(HEADS):
            d.w1[h] = self.tensors[f"{head}_w1"].data_ptr()
            d.b1[h] = self.tensors[f"{head}_b1"].data_ptr()
            d.w2[h] = self.tensors[f"{head}_w2"].data_ptr()
            d.b2[h] = self.tensors[f"{head}_b2"].data_ptr()
        d.n = self.n
        return d


def grads_abi(grads: dict[str, torch.Tensor]) -> VsxDecoderGrads:
    g = VsxDecoderGrads()
    for h, head in enumerate(HEADS):
        g.w1[h] = grads[f"{head}_w1"].data_ptr()
        g.b1[h] = grads[f"{head}_b1"].data_ptr()
        g.w2[h] = grads[f"{head}_w2"].data_ptr()
        g.b2[h] = grads[f"{head}_b2"].data_ptr()
    return g


def params_equal(a: DecoderParams, b: DecoderParams) -> bool:
    if a.n != b.n or a.tensors.keys() != b.tensors.keys():
        return False
    return all(torch.equal(a.tensors[k], b.tensors[k]) for k in a.tensors)


def quat_to_rotmat_t(q: torch.Tensor) -> torch.Tensor:
    w, x, y, z = q.unbind(-1)
    m = [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]
    return torch.stack(m, -1).reshape(*q.shape[:-1], 3, 3)


@dataclass
class AnchorState:
    """Flat (level-major) per-anchor parameters on the device.

    The trainer's live state; ``scales`` of the reference are exp(log_scales)
    evaluated in float64 inside the kernels.
    """

    emb: torch.Tensor          # (A, 32) f32
    log_scales: torch.Tensor   # (A, 3) f32
    offsets: torch.Tensor      # (A, n, 3) f32

    @classmethod
    def from_scene(cls, scene) -> "AnchorState":
        require_cuda()
        f32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
        return cls(f32(scene.flat("embeddings")), f32(np.log(scene.flat("scales"))),
                   f32(scene.flat("offsets")))


class GaussianBatch:
    """Decoded gaussians in canonical order; tensors live on the device.

    ``level``, ``voxel_index``, ``owner`` and ``gid`` (numpy bookkeeping in
    the reference, ``decoder.py:117-139``) are materialised lazily on access
    so the hot loop never synchronises for them.
    """

    def __init__(self, means, opacities, colors, scales, quats, normals, active=None, n=1,
                 level_bases=None, owner_of_anchor=None, leaves=None, decoded=None):
        self.means, self.opacities, self.colors = means, opacities, colors
        self.scales, self.quats, self.normals = scales, quats, normals
        self._active, self._n = active, n
        self._level_bases = level_bases
        self._owner = owner_of_anchor
        self.leaves = leaves
        self.decoded = decoded

    @property
    def count(self) -> int:
        return int(self.means.shape[0])

    def _anchor_ids(self) -> np.ndarray:
        if self._active is None:
            return np.arange(self.count, dtype=np.int64)
        return self._active.cpu().numpy().astype(np.int64)

    @property
    def gid(self) -> np.ndarray:
        a = self._anchor_ids()
        if self._active is None:
            return a
        return (a[:, None] * self._n + np.arange(self._n)).reshape(-1)

    @property
    def level(self) -> np.ndarray:
        if self._active is None:
            return np.zeros(self.count, np.int32)
        a = self._anchor_ids()
        lv = np.searchsorted(self._level_bases, a, side="right") - 1
        return np.repeat(lv.astype(np.int32), self._n)

    @property
    def voxel_index(self) -> np.ndarray:
        if self._active is None:
            return np.arange(self.count, dtype=np.int64)
        a = self._anchor_ids()
        lv = np.searchsorted(self._level_bases, a, side="right") - 1
        return np.repeat(a - self._level_bases[lv], self._n)

    @property
    def owner(self) -> np.ndarray:
        if self._active is None or self._owner is None:
            return np.zeros(self.count, np.int32)
        return np.repeat(self._owner[self._anchor_ids()], self._n)


class _DecodeFn(torch.autograd.Function):
    """Autograd bridge: forward = vsx_decode_fwd, backward = vsx_decode_bwd."""

    @staticmethod
    def forward(ctx, meta, emb, log_scales, offsets, *weights):
        params, active, centers, view, lod_ref, max_scale, status = meta
        dec = _decode(params.abi(), params.n, active, centers, emb, log_scales, offsets, view,
                      lod_ref, max_scale, status, keep_cache=True)
        ctx.meta = meta
        ctx.dec = dec
        ctx.save_for_backward(emb, log_scales, offsets)
        return dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal

    @staticmethod
    def backward(ctx, gm, go, gc, gs, gq, gn):
        params, active, centers, view, lod_ref, max_scale, _ = ctx.meta
        emb, log_scales, offsets = ctx.saved_tensors
        dec: Decoded = ctx.dec
        z = lambda t, like: (t if t is not None else torch.zeros_like(like)).float().contiguous()  # noqa: E731
        gm, go, gc = z(gm, dec.means), z(go, dec.opacity), z(gc, dec.color)
        gs, gq, gn = z(gs, dec.scale), z(gq, dec.quat), z(gn, dec.normal)
        d_emb = torch.zeros_like(emb)
        d_ls = torch.zeros_like(log_scales)
        d_off = torch.zeros_like(offsets)
        d_w = {k: torch.zeros_like(v) for k, v in params.tensors.items()}
        decoder_backward_into(params, d_w, active, centers, emb, log_scales, offsets, view,
                              lod_ref, max_scale, dec, gm, go, gc, gs, gq, gn, d_emb, d_ls, d_off)
        return (None, d_emb, d_ls, d_off, *[d_w[k] for k in params.param_names(params.n)])


def decoder_backward_into(params, d_w, active, centers, emb, log_scales, offsets, view, lod_ref,
                          max_scale, dec: Decoded, gm, go, gc, gs, gq, gn, d_emb, d_ls, d_off):
    """Accumulate (+=) K8 gradients into caller-owned buffers."""
    na = int(active.numel())
    if na == 0:
        return
    lib = _lib.load()
    wp, wb = workspace().get(lib.vsx_decode_bwd_ws_bytes(params.n, na))
    call("vsx_decode_bwd", params.abi(), grads_abi(d_w), ptr(active), na, ptr(centers), ptr(emb),
         ptr(log_scales), ptr(offsets), view.to_abi(), lod_ref, max_scale, ptr(dec.cache_h),
         ptr(dec.cache_o), ptr(dec.scale), ptr(dec.quat), ptr(gm), ptr(go), ptr(gc), ptr(gs),
         ptr(gq), ptr(gn), ptr(d_emb), ptr(d_ls), ptr(d_off), wp, wb, stream())


def _anchor_source(scene, state):
    if state is None:
        return AnchorState.from_scene(scene)
    if isinstance(state, AnchorState):
        return state
    raise InvalidInput("state must be an AnchorState (flat device anchors) or None")


def decode_active(params: DecoderParams, scene, view: CameraView, state=None,
                  keep_graph: bool = False, validate: bool = True) -> GaussianBatch:
    """Decode every voxel active for ``view`` (``decoder.py:210-250``)."""
    ds = device_scene_for(scene)
    active = ds.active(view)
    return decode_indices(params, scene, active, view, state, keep_graph, validate)


def decode_indices(params: DecoderParams, scene, active: torch.Tensor, view: CameraView,
                   state=None, keep_graph=False, validate=True) -> GaussianBatch:
    ds = device_scene_for(scene)
    src = _anchor_source(scene, state)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    owner = np.concatenate([lv.owner for lv in scene.levels]) if scene.levels else None
    if keep_graph:
        meta = (params, active, ds.centers, view, ds.lod_ref, ds.max_scale, status)
        w = [params.tensors[k] for k in params.param_names(params.n)]
        outs = _DecodeFn.apply(meta, src.emb, src.log_scales, src.offsets, *w)
        batch = GaussianBatch(*outs, active=active, n=params.n, level_bases=ds.level_bases,
                              owner_of_anchor=owner)
    else:
        dec = _decode(params.abi(), params.n, active, ds.centers, src.emb, src.log_scales,
                      src.offsets, view, ds.lod_ref, ds.max_scale, status, keep_cache=False)
        batch = GaussianBatch(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal,
                              active=active, n=params.n, level_bases=ds.level_bases,
                              owner_of_anchor=owner, decoded=dec)
    if validate:
        check_status(status, "decode")
    return batch


def decode_inputs(centers: torch.Tensor, embeddings: torch.Tensor, cam_center,
                  lod_ref: float) -> torch.Tensor:
    """The (V, 36) decoder input block [emb | d/ref | (c - cam)/d], d clamped
    at 1e-12 (``decoder.py:142-147``), on the device.

    API compatibility only: the training path never materialises it (K2
    assembles each row in registers from the anchor arrays)."""
    require_cuda()
    c = torch.as_tensor(centers, device="cuda", dtype=torch.float64)
    rel = c - torch.as_tensor(np.asarray(cam_center, np.float64), device="cuda")
    dist = torch.linalg.norm(rel, dim=-1, keepdim=True).clamp_min(1e-12)
    emb = torch.as_tensor(embeddings, device="cuda")
    return torch.cat([emb.double(), dist / lod_ref, rel / dist], dim=-1).to(emb.dtype)


def decode_arrays(params: DecoderParams, centers, embeddings, scales, offsets,
                  view: CameraView, lod_ref: float, max_scale: float) -> dict:
    """Decode V voxels of explicit state into (V, n, ...) gaussian attributes
    (``decoder.py:150-180``) through the K2 kernel.

    ``scales`` is the voxel scale triple l_v (positive); the kernel takes log
    scales, so it is passed as log(l_v) (differentiably when it requires
    grad). Graph-connected when any input or weight requires grad, with the
    K8 kernel as its backward."""
    require_cuda()
    c = torch.as_tensor(centers, device="cuda", dtype=torch.float64).reshape(-1, 3).contiguous()
    v, n = int(c.shape[0]), params.n
    f32 = lambda x: torch.as_tensor(x, device="cuda").float()  # noqa: E731
    emb = f32(embeddings).reshape(v, -1).contiguous()
    log_s = torch.log(f32(scales).reshape(v, 3)).contiguous()
    off = f32(offsets).reshape(v, n, 3).contiguous()
    active = torch.arange(v, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    w = [params.tensors[k] for k in params.param_names(n)]
    if torch.is_grad_enabled() and any(t.requires_grad for t in [emb, log_s, off, *w]):
        meta = (params, active, c, view, float(lod_ref), float(max_scale), status)
        outs = _DecodeFn.apply(meta, emb, log_s, off, *w)
    else:
        dec = _decode(params.abi(), n, active, c, emb, log_s, off, view, float(lod_ref),
                      float(max_scale), status, keep_cache=False)
        outs = (dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal)
    check_status(status, "decode_arrays")
    means, opac, col, scl, quat, nrm = outs
    return {"means": means.reshape(v, n, 3), "opacities": opac.reshape(v, n),
            "colors": col.reshape(v, n, 3), "scales": scl.reshape(v, n, 3),
            "quats": quat.reshape(v, n, 4), "normals": nrm.reshape(v, n, 3)}


def decode_level(params: DecoderParams, scene, level: int, indices: np.ndarray,
                 view: CameraView, max_scale: float | None = None, state=None,
                 keep_graph: bool = False) -> dict | None:
    """Decode given voxel indices of one level; tensors shaped (V, n, …)."""
    indices = np.asarray(indices, np.int64)
    if indices.size == 0:
        return None
    base = int(scene.level_bases[level])
    active = torch.as_tensor((indices + base).astype(np.int32)).cuda()
    b = decode_indices(params, scene, active, view, state, keep_graph, validate=False)
    v, n = indices.size, params.n
    return {"means": b.means.reshape(v, n, 3), "opacities": b.opacities.reshape(v, n),
            "colors": b.colors.reshape(v, n, 3), "scales": b.scales.reshape(v, n, 3),
            "quats": b.quats.reshape(v, n, 4), "normals": b.normals.reshape(v, n, 3)}


def decoder_backward(outputs: dict, upstream: dict, leaves: dict) -> dict:
    """Pull cotangents on decoded attributes back to leaves (``decoder.py:267-292``)."""
    outs, cots, seen = [], [], 0
    for k, out in outputs.items():
        if k in upstream and upstream[k] is not None:
            seen += 1
            if out.requires_grad:
                outs.append(out)
                cots.append(torch.as_tensor(np.asarray(upstream[k]) if not torch.is_tensor(upstream[k])
                                            else upstream[k]).to(out.device, out.dtype)
                            .reshape(out.shape))
    if seen == 0:
        raise InvalidInput("no upstream gradients supplied")
    if not outs:
        raise StateError("decode was not run with keep_graph=True")
    names = list(leaves)
    grads = torch.autograd.grad(outs, [leaves[n] for n in names], grad_outputs=cots,
                                retain_graph=True, allow_unused=True)
    return {n: (g if g is not None else torch.zeros_like(leaves[n])) for n, g in zip(names, grads)}


def sync_params(worker_grads: list[dict]) -> dict:
    """Mean of per-worker gradient sets in worker-id order (``decoder.py:295-312``)."""
    if not worker_grads:
        raise ProtocolError("sync called with no participants")
    keys = list(worker_grads[0])
    for i, g in enumerate(worker_grads):
        if list(g) != keys:
            raise ProtocolError(f"worker {i} gradient keys differ")
        for k in keys:
            if g[k].shape != worker_grads[0][k].shape:
                raise ProtocolError(f"worker {i} gradient shape differs for {k}")
    out = {}
    for k in keys:
        acc = worker_grads[0][k].clone()
        for g in worker_grads[1:]:
            acc = acc + g[k]
        out[k] = acc / len(worker_grads)
    return out
