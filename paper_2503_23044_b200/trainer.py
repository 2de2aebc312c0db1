"""Batch-level multi-view training step on the B200 (``voxsplat/trainer.py``).

``TrainState`` keeps every learnable tensor in ONE flat float32 device buffer
(decoder tensors, then per-anchor embeddings, log-scales, offsets, level-
major), with matching flat gradient and Adam-moment buffers, so the whole
optimizer step is a single ``vsx_adam`` launch (K10).

``train_step`` runs, per view: K1 cull -> K2 decode -> K3 project + radix
sort -> K4 bin -> K5 composite -> K9 loss with fused cotangents -> K6
composite backward -> K7 projection backward -> K8 decode backward
(accumulating into the flat gradient). The batch loss is a sum of per-view
terms, so each view's backward runs right after its forward and nothing per
view outlives it. Then one Adam launch. Semantics follow
``trainer.py:258-376`` (RGB L1 always; Eq. 9 depth term weighted by the stage
schedule when priors are given).
"""

from __future__ import annotations

import contextlib
from types import SimpleNamespace
import ctypes
import json
import threading
import time
import os
from dataclasses import dataclass, fields

import numpy as np
import torch

from . import device as D
from ._lib import VsxLossDesc, call, ptr, stream
from .decoder import AnchorState, DecoderParams, decoder_backward_into
from .errors import InvalidInput, NumericalError
from .geometry import CameraView
from .partition import PatchCostModel, assign_voxels, balance_report, schedule_patches

ADAM_EPS = 1e-15


@dataclass
class TrainConfig:
    total_steps: int = 2000
    batch_size: int = 4
    workers: int = 1
    seed: int = 0
    step2_start: int = 800
    step3_start: int = 1400
    lr_decoder: float = 2e-3
    lr_embeddings: float = 5e-3
    lr_offsets: float = 1e-2
    lr_scales: float = 5e-3
    lr_final_factor: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    growth_threshold: float = 2e-4
    growth_window: int = 100
    growth_stop: int = 1000
    w3_max: float = 0.2
    tau_depth: float = 1.0
    geo_patches: int = 64
    geo_patch_half: int = 3
    init_scale_fraction: float = 0.125
    # extension: weight of the normal-prior L1 (0 = reference objective)
    normal_weight: float = 0.0
    # bitwise run-to-run reproducible sums: the compositor's per-splat
    # gradients and the loss sums are reduced in a fixed order instead of by
    # float atomics (vsx_raster_grad_reduce / vsx_reduce_partials), and the
    # sharded step's decoder all-reduce becomes an all-gather + ordered sum.
    # The Eq. 10 NCC term keeps its atomics.
    deterministic: bool = False
    log_every: int = 10
    eval_every: int = 0
    checkpoint_every: int = 0

    def validate(self) -> None:
        if self.total_steps < 1:
            raise InvalidInput("total_steps must be >= 1")
        for name in ("step2_start", "step3_start"):
            if not 0 <= getattr(self, name) <= self.total_steps:
                raise InvalidInput(f"{name} must lie in [0, total_steps]")
        if self.batch_size < 1 or self.workers < 1 or self.growth_window < 1:
            raise InvalidInput("batch_size, workers and growth_window must be >= 1")
        if not 0 < self.lr_final_factor <= 1:
            raise InvalidInput("lr_final_factor must be in (0, 1]")
        for name in ("lr_decoder", "lr_embeddings", "lr_offsets", "lr_scales"):
            if getattr(self, name) <= 0:
                raise InvalidInput(f"{name} must be positive")
        if not 0 < self.init_scale_fraction <= 3:
            raise InvalidInput("init_scale_fraction must be in (0, 3]")

    @classmethod
    def from_dict(cls, data: dict) -> "TrainConfig":
        bad = set(data) - {f.name for f in fields(cls)}
        if bad:
            raise InvalidInput(f"unknown train config keys: {sorted(bad)}")
        cfg = cls(**data)
        cfg.validate()
        return cfg


def weight_schedule(step: int, cfg: TrainConfig) -> tuple[float, float]:
    w2 = 0.0
    if step >= cfg.step2_start and cfg.total_steps > cfg.step2_start:
        w2 = 1.0 - (step - cfg.step2_start) / (cfg.total_steps - cfg.step2_start)
    w3 = 0.0
    if step >= cfg.step3_start and cfg.total_steps > cfg.step3_start:
        w3 = cfg.w3_max * (step - cfg.step3_start) / (cfg.total_steps - cfg.step3_start)
    return w2, w3


def cosine_lr(step: int, base: float, cfg: TrainConfig) -> float:
    lo = base * cfg.lr_final_factor
    return lo + 0.5 * (base - lo) * (1.0 + np.cos(np.pi * step / cfg.total_steps))


@dataclass
class StepReport:
    step: int
    total: float
    rgb: float
    depth: float
    geo: float
    w2: float
    w3: float
    lr: float
    supervised_depth_px: int
    geo_pairs: int
    geo_patches: int
    gaussians: int
    transfer_bytes: int
    imbalance: float
    max_tile_splats: int
    seconds: float
    grown: int = 0
    intersections: int = 0
    normal: float = 0.0
    live_pairs: int = 0     # (pixel, splat) pairs composited = sum of per-pixel live counts

    def to_json(self) -> str:
        return json.dumps({
            "step": self.step, "total": self.total, "rgb": self.rgb, "depth": self.depth,
            "geo": self.geo, "w2": self.w2, "w3": self.w3, "lr": self.lr,
            "depth_px": self.supervised_depth_px, "geo_pairs": self.geo_pairs,
            "geo_patches": self.geo_patches, "gaussians": self.gaussians,
            "transfer_bytes": self.transfer_bytes, "imbalance": self.imbalance,
            "max_tile_splats": self.max_tile_splats, "seconds": self.seconds,
            "grown": self.grown})


def _pad4(n: int) -> int:
    return (n + 3) // 4 * 4


class FlatParams:
    """One flat float32 buffer (+ grad, m, v) carved into named views."""

    def __init__(self, shapes: list[tuple[str, tuple]], groups: dict[str, str]):
        self.layout = {}
        off = 0
        self.group_spans: dict[str, list[int]] = {}
        for name, shape in shapes:
            n = int(np.prod(shape)) if shape else 1
            self.layout[name] = (off, shape)
            g = groups[name]
            span = self.group_spans.setdefault(g, [off, off])
            span[1] = off + _pad4(n)
            off += _pad4(n)
        self.size = off
        dev = "cuda"
        self.param = torch.zeros(self.size, dtype=torch.float32, device=dev)
        self.grad = torch.zeros_like(self.param)
        self.m = torch.zeros_like(self.param)
        self.v = torch.zeros_like(self.param)

    def view(self, buf: torch.Tensor, name: str) -> torch.Tensor:
        off, shape = self.layout[name]
        n = int(np.prod(shape)) if shape else 1
        return buf[off:off + n].view(shape)

    def segments(self, order: list[str]) -> tuple[list[int], list[str]]:
        """Contiguous [begin, end) per group in buffer order (for vsx_adam)."""
        spans = sorted(((self.group_spans[g][0], self.group_spans[g][1], g) for g in order))
        begins = [s[0] for s in spans] + [spans[-1][1]]
        for (b0, e0, _), (b1, _, _) in zip(spans, spans[1:]):
            if e0 != b1:
                raise InvalidInput("flat parameter groups are not contiguous")
        return begins, [s[2] for s in spans]


class TrainState:
    """Scene mirrors, the decoder replica and Adam state, all on the device."""

    def __init__(self, scene, cfg: TrainConfig):
        cfg.validate()
        D.require_cuda()
        self.scene = scene
        self.cfg = cfg
        self.step = 0
        self.rng = np.random.default_rng(cfg.seed)
        n = scene.offsets_per_voxel
        A = scene.total_voxels
        self.n = n
        init = DecoderParams.init_arrays(
            n, seed=cfg.seed,
            scale_bias=float(np.log(cfg.init_scale_fraction * scene.base_voxel_size)))
        names = DecoderParams.param_names(n)
        self.flat = self._alloc_flat(A)
        with torch.no_grad():
            for k in names:
                self.flat.view(self.flat.param, f"dec/{k}").copy_(
                    torch.as_tensor(init[k], dtype=torch.float32))
            self.flat.view(self.flat.param, "emb").copy_(
                torch.as_tensor(scene.flat("embeddings"), dtype=torch.float32))
            self.flat.view(self.flat.param, "log_scales").copy_(
                torch.as_tensor(np.log(scene.flat("scales")), dtype=torch.float32))
            self.flat.view(self.flat.param, "offsets").copy_(
                torch.as_tensor(scene.flat("offsets"), dtype=torch.float32))
        self._bind_views()
        self.assignment = assign_voxels(scene, cfg.workers)
        self.dscene = D.device_scene_for(scene)
        self._image_cache: dict = {}
        # per-patch EMA cost model of the simulated multi-worker schedule
        # (trainer.py:264-268, 355-364); only consulted when cfg.workers > 1
        self.cost_model = PatchCostModel()
        self._inflight = None
        # growth pressure (trainer.py:341-349): per anchor, sum and count of
        # the decoded-position gradient norms of its gaussians (flat, level-major)
        self.grow_sum_flat = torch.zeros(A, dtype=torch.float64, device="cuda")
        self.grow_cnt_flat = torch.zeros(A, dtype=torch.float64, device="cuda")
        self.grow_events: list[dict] = []

    def _alloc_flat(self, A: int) -> "FlatParams":
        n = self.n
        dec_shapes = DecoderParams.shapes(n)
        names = DecoderParams.param_names(n)
        shapes = [(f"dec/{k}", dec_shapes[k]) for k in names]
        shapes += [("emb", (A, 32)), ("log_scales", (A, 3)), ("offsets", (A, n, 3))]
        groups = {f"dec/{k}": "dec" for k in names}
        groups.update({"emb": "emb", "log_scales": "log_scales", "offsets": "offsets"})
        return FlatParams(shapes, groups)

    def _bind_views(self) -> None:
        names = DecoderParams.param_names(self.n)
        self.params = DecoderParams(self.n, {k: self.flat.view(self.flat.param, f"dec/{k}")
                                             for k in names})
        self.dgrads = {k: self.flat.view(self.flat.grad, f"dec/{k}") for k in names}
        self.replicas = [self.params]
        self.anchors = AnchorState(self.flat.view(self.flat.param, "emb"),
                                   self.flat.view(self.flat.param, "log_scales"),
                                   self.flat.view(self.flat.param, "offsets"))
        self.anchor_grads = AnchorState(self.flat.view(self.flat.grad, "emb"),
                                        self.flat.view(self.flat.grad, "log_scales"),
                                        self.flat.view(self.flat.grad, "offsets"))

    def _per_level(self, flat: torch.Tensor) -> dict:
        b = self.scene.level_bases
        host = flat.cpu().numpy()
        return {k: host[int(b[k]):int(b[k + 1])].copy() for k in range(self.scene.lod_count)}

    @property
    def grow_sum(self) -> dict:
        """Reference-shaped per-level growth sums (host copies)."""
        return self._per_level(self.grow_sum_flat)

    @property
    def grow_cnt(self) -> dict:
        return self._per_level(self.grow_cnt_flat)

    def _insert_anchors(self, old_bases: np.ndarray, additions: dict) -> None:
        """Re-lay the flat buffers after growth: every level keeps its rows and
        gets its new anchors appended (level-major); new Adam moments are 0."""
        new = self._alloc_flat(self.scene.total_voxels)
        old = self.flat
        nb = self.scene.level_bases
        with torch.no_grad():
            for name in old.layout:
                if name.startswith("dec/"):
                    for b_old, b_new in ((old.param, new.param), (old.m, new.m), (old.v, new.v)):
                        new.view(b_new, name).copy_(old.view(b_old, name))
            for name, key in (("emb", 0), ("log_scales", 1), ("offsets", 2)):
                for k in range(self.scene.lod_count):
                    lo, hi = int(old_bases[k]), int(old_bases[k + 1])
                    dst = int(nb[k])
                    for b_old, b_new in ((old.param, new.param), (old.m, new.m),
                                         (old.v, new.v)):
                        new.view(b_new, name)[dst:dst + hi - lo].copy_(
                            old.view(b_old, name)[lo:hi])
                    if k in additions:
                        arr = torch.as_tensor(additions[k][key], dtype=torch.float32)
                        new.view(new.param, name)[dst + hi - lo:int(nb[k + 1])].copy_(arr)
        self.flat = new
        self._bind_views()
        self.dscene = D.device_scene_for(self.scene)
        self._image_cache = {}

    # -- reference-compatible views ---------------------------------------
    @property
    def moments(self) -> dict:
        out = {}
        for name in self.flat.layout:
            out[name] = (self.flat.view(self.flat.m, name), self.flat.view(self.flat.v, name))
        return out

    def barrier_check(self) -> None:
        """Single replica per process; cross-rank equality is checked by dist.py."""

    def decode_state(self) -> AnchorState:
        return self.anchors

    def sync_to_scene(self) -> None:
        A_bases = self.scene.level_bases
        emb = self.anchors.emb.double().cpu().numpy()
        ls = self.anchors.log_scales.double().cpu().numpy()
        off = self.anchors.offsets.double().cpu().numpy()
        for k, lv in enumerate(self.scene.levels):
            lo, hi = int(A_bases[k]), int(A_bases[k + 1])
            lv.embeddings = emb[lo:hi].copy()
            lv.scales = np.exp(ls[lo:hi])
            lv.offsets = off[lo:hi].copy()

    def lrs(self) -> dict[str, float]:
        c = self.cfg
        return {"dec": cosine_lr(self.step, c.lr_decoder, c),
                "emb": cosine_lr(self.step, c.lr_embeddings, c),
                "log_scales": cosine_lr(self.step, c.lr_scales, c),
                "offsets": cosine_lr(self.step, c.lr_offsets, c)}

    def adam(self, guard: torch.Tensor | None = None) -> None:
        """One fused Adam launch over every parameter group (K10); with a
        device int32 ``guard`` the update is skipped on the device when it is
        nonzero."""
        begins, order = self.flat.segments(["dec", "emb", "log_scales", "offsets"])
        lrs = self.lrs()
        nseg = len(order)
        seg = (ctypes.c_int64 * (nseg + 1))(*begins)
        lr = (ctypes.c_double * nseg)(*[lrs[g] for g in order])
        f = self.flat
        if guard is not None:
            call("vsx_adam_guarded", ptr(f.param), ptr(f.grad), ptr(f.m), ptr(f.v), nseg, seg,
                 lr, self.cfg.beta1, self.cfg.beta2, ADAM_EPS, self.step, ptr(guard), stream())
            return
        call("vsx_adam", ptr(f.param), ptr(f.grad), ptr(f.m), ptr(f.v), nseg, seg, lr,
             self.cfg.beta1, self.cfg.beta2, ADAM_EPS, self.step, stream())


def make_state(scene, cfg: TrainConfig) -> TrainState:
    return TrainState(scene, cfg)


def _to_device_image(x, shape) -> torch.Tensor:
    t = x if torch.is_tensor(x) else torch.as_tensor(np.asarray(x))
    t = t.to(device="cuda", dtype=torch.float32, non_blocking=True).contiguous()
    if tuple(t.shape) != tuple(shape):
        raise InvalidInput(f"image shape mismatch {tuple(t.shape)} vs {tuple(shape)}")
    return t


def _prior_arrays(e):
    if e is None:
        return None
    if isinstance(e, tuple):
        return e
    return e.values, e.valid


@dataclass
class ViewWork:
    """Per-view device intermediates kept for inspection (tests / bench)."""

    active: torch.Tensor
    decoded: D.Decoded
    projected: D.Projected
    bins: D.Bins
    raster: D.Raster
    grad_splat: torch.Tensor
    grad_gauss: dict


class GpuTimer:
    """CUDA-event spans on the current stream, summed per stage name."""

    def __init__(self) -> None:
        self.spans: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []

    @contextlib.contextmanager
    def span(self, name: str):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        try:
            yield
        finally:
            b.record()
            self.spans.append((name, a, b))

    def totals_ms(self) -> dict[str, float]:
        torch.cuda.synchronize()
        out: dict[str, float] = {}
        for name, a, b in self.spans:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out

    def counts(self) -> dict[str, int]:
        out: dict[str, int] = {}
        for name, _, _ in self.spans:
            out[name] = out.get(name, 0) + 1
        return out


_NULL = contextlib.nullcontext()


def _span(timer, name):
    return timer.span(name) if timer is not None else _NULL


def _mask_u8(v, shape) -> torch.Tensor:
    t = v if torch.is_tensor(v) else torch.as_tensor(np.asarray(v))
    t = t.to(device="cuda", dtype=torch.uint8, non_blocking=True).contiguous()
    if tuple(t.shape) != tuple(shape):
        raise InvalidInput(f"mask shape mismatch {tuple(t.shape)} vs {tuple(shape)}")
    return t


# Side streams of the per-view pipeline, one set per host thread (a host
# thread drives one device; the sort/scan scratch buffers are keyed by stream,
# so threads must not share streams).
_STREAMS = threading.local()


def _side_stream(name: str, priority: int = 0) -> torch.cuda.Stream:
    st = getattr(_STREAMS, name, None)
    if st is None or st.device != torch.device("cuda", torch.cuda.current_device()):
        st = torch.cuda.Stream(priority=priority)
        setattr(_STREAMS, name, st)
    return st
# VSX_TRACE=1: host timestamps of the step's phases (diagnosing host stalls)
_TRACE = os.environ.get("VSX_TRACE") == "1"
TRACE_LOG: list = []


def reserve_stream_pools(nbytes: int) -> None:
    """Grow the caching allocator's pool of every pipeline stream by nbytes.

    Blocks are cached per stream, so head-room reserved on one stream does
    not serve another. Mapping new device memory inside a step can stall the
    host for as long as the queued GPU work (tens of ms); a long-running
    trainer (or a benchmark) calls this once after warm-up."""
    cur = torch.cuda.current_stream()
    streams = [cur]
    if _pipeline_enabled():
        streams += [_front_stream(), _tail_stream()]
    if getattr(_STREAMS, "copy", None) is not None:
        streams.append(_STREAMS.copy)
    for st in streams:
        with torch.cuda.stream(st):
            pad = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            del pad
    torch.cuda.synchronize()


def _tr(label):
    if _TRACE:
        TRACE_LOG.append((label, time.perf_counter()))


def _front_stream() -> torch.cuda.Stream:
    return _side_stream("front", priority=-1)  # ahead of the compositor's CTAs


def _tail_stream() -> torch.cuda.Stream:
    return _side_stream("tail")


def _pipeline_enabled() -> bool:
    """VSX_PIPELINE=0 runs every view's stages back to back on one stream (A/B)."""
    import os
    return os.environ.get("VSX_PIPELINE", "1") != "0"


class _InputStager:
    """Per-view targets/priors moved to the device on a copy stream.

    All host->device copies of the step are issued up front (non-blocking
    from pinned host memory), one event per view; view v's compute waits only
    for its own inputs, so the copies of later views overlap the compute of
    earlier ones. CUDA inputs pass through untouched.
    """

    def __init__(self, views, images, priors, have, normal_priors, have_n, only=None,
                 prefetch=False):
        cur = torch.cuda.current_stream()
        cs = _side_stream("copy")
        if not prefetch:
            # (a prefetch depends on nothing but host memory and fresh blocks:
            # it may run under the current step's compute)
            cs.wait_stream(cur)
        self.items, self.events = [], []
        with torch.cuda.stream(cs):
            for vi, view in enumerate(views):
                if only is not None and vi not in only:   # rendered by another rank
                    self.items.append((None,) * 5)
                    self.events.append(None)
                    continue
                H, W = view.height, view.width
                gt = _to_device_image(images[vi], (H, W, 3))
                pd = pv = pn = pnv = None
                if vi in have:
                    pd = _to_device_image(priors[vi][0], (H, W))
                    pv = _mask_u8(priors[vi][1], (H, W))
                if vi in have_n:
                    pn = _to_device_image(normal_priors[vi][0], (H, W, 3))
                    pnv = _mask_u8(normal_priors[vi][1], (H, W))
                for t in (gt, pd, pv, pn, pnv):
                    if t is not None:
                        t.record_stream(cur)  # freed only after the compute stream used it
                ev = torch.cuda.Event()
                ev.record(cs)
                self.items.append((gt, pd, pv, pn, pnv))
                self.events.append(ev)

    def get(self, vi):
        if self.events[vi] is not None:
            torch.cuda.current_stream().wait_event(self.events[vi])
        return self.items[vi]


class StagedInputs:
    """A batch's targets and priors already on their way to the device.

    The host->device copies (pinned host memory, the copy stream) are issued
    when this is built, so building step k+1's inputs before calling
    ``train_step`` for step k overlaps them with step k's compute — the
    double-buffered input pipeline of a training loop. Pass it as
    ``train_step``'s ``images``; its ``enhanced`` / ``normal_priors`` are
    used (priors the step's schedule leaves unused are ignored).
    """

    def __init__(self, views: list[CameraView], images: list, enhanced: list | None = None,
                 normal_priors: list | None = None):
        B = len(views)
        if B == 0 or len(images) != B:
            raise InvalidInput("views and images must be equal length and non-empty")
        self.views, self.images = views, images
        self.enhanced, self.normal_priors = enhanced, normal_priors
        priors = [_prior_arrays(e) for e in enhanced] if enhanced is not None else None
        have = [i for i in range(B) if priors is not None and priors[i] is not None]
        have_n = [i for i in range(B) if normal_priors is not None and normal_priors[i] is not None]
        self.stager = _InputStager(views, images, priors, have, normal_priors, have_n,
                                   prefetch=True)

    def __len__(self) -> int:
        return len(self.images)


def train_step(state: TrainState, views: list[CameraView], images: list,
               enhanced: list | None = None, keep: list | None = None,
               normal_priors: list | None = None, timer: GpuTimer | None = None) -> StepReport:
    """One optimisation step over a batch of views (``trainer.py:258-376``).

    ``enhanced`` holds per-view depth priors (EnhancedDepthMap or (depth,
    valid)) for the Eq. 9 term, weighted by the stage schedule.
    ``normal_priors`` (optional, (normals, valid) per view) add the normal
    term of the RGB-D-N objective with weight ``cfg.normal_weight`` (an
    extension: the reference supervises normals only through the depth
    quotient and Eq. 10). Images/priors may be host arrays or CUDA tensors.
    """
    cfg = state.cfg
    t0 = time.perf_counter()
    B = len(views)
    staged = images if isinstance(images, StagedInputs) else None
    if staged is not None:
        if len(staged.views) != B:
            raise InvalidInput("StagedInputs built for another batch")
        images, enhanced, normal_priors = staged.images, staged.enhanced, staged.normal_priors
    if B == 0 or len(images) != B:
        raise InvalidInput("views and images must be equal length and non-empty")
    w2, w3 = weight_schedule(state.step, cfg)
    priors = [_prior_arrays(e) for e in enhanced] if enhanced is not None else None
    use_depth = w2 > 0 and priors is not None and any(p is not None for p in priors)
    have = [i for i in range(B) if use_depth and priors[i] is not None]
    wn = float(getattr(cfg, "normal_weight", 0.0))
    use_normal = wn > 0 and normal_priors is not None
    have_n = [i for i in range(B) if use_normal and normal_priors[i] is not None]
    ds = state.dscene
    params = state.params
    st = state.flat
    st.grad.zero_()
    dev = "cuda"
    sums = torch.zeros((B, 3), dtype=torch.float64, device=dev)     # rgb, depth, normal |d|
    counts = torch.zeros((B, 2), dtype=torch.int32, device=dev)     # depth px, normal px
    rgb_acc, dep_sum, nrm_sum = sums[:, 0], sums[:, 1], sums[:, 2]
    dep_cnt, nrm_cnt = counts[:, 0], counts[:, 1]
    tile_max = torch.zeros(1, dtype=torch.int32, device=dev)   # longest tile list (u32)
    live = torch.zeros((), dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    gaussians = 0
    isects = 0
    anchors, agrads = state.anchors, state.anchor_grads
    stager = staged.stager if staged is not None else \
        _InputStager(views, images, priors, have, normal_priors, have_n)
    book = _WorkerBook(state, views) if cfg.workers > 1 else None
    main = torch.cuda.current_stream()
    # Three-stream software pipeline over the views: the front end of view v+1
    # (cull, decode, project + sort, binning: small, latency-bound kernels and
    # the host reads of their counts) runs on a high-priority side stream, and
    # the projection/decoder backward of view v-1 on a tail stream, while the
    # compositor of view v runs on the main stream. Per-view
    # device buffers stay referenced until the end-of-step sync, so the caching
    # allocator never recycles a side-stream block the main stream still reads.
    fs = _front_stream() if _pipeline_enabled() else main
    ts = _tail_stream() if _pipeline_enabled() else main
    # the decoder weight image (3xTF32 fragments) once per step, not per view
    dimg = D.decoder_image(params.abi(), params.n) if D.use_tensor_cores(params.n) else None
    fs.wait_stream(main)
    ts.wait_stream(main)
    hold = []
    fronts = {}

    def front(vi):
        view = views[vi]
        _tr(f"front{vi}")
        with torch.cuda.stream(fs):
            with _span(timer, "cull"):
                active = ds.active(view)
            with _span(timer, "decode_fwd"):
                dec = D.decode(params.abi(), params.n, active, ds.centers, anchors.emb,
                               anchors.log_scales, anchors.offsets, view, ds.lod_ref,
                               ds.max_scale, status, keep_cache=True, img=dimg)
            with _span(timer, "project_sort"):
                P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal,
                              view, status)
            with _span(timer, "bin_sort"):
                Bn = D.bin_tiles(P, view.width, view.height)
            call("vsx_tile_max_len", ptr(Bn.tile_offsets), Bn.tiles_x * Bn.tiles_y,
                 ptr(tile_max), stream())
            ev = torch.cuda.Event()
            ev.record(fs)
        fronts[vi] = (active, dec, P, Bn, ev)
        _tr(f"front{vi}_done")

    def loss_desc(vi, extra=None):
        view = views[vi]
        gt, pd, pv, pn, pnv = stager.get(vi)
        if vi not in have:          # a prefetched prior the schedule does not use
            pd = pv = None
        if vi not in have_n:
            pn = pnv = None
        ex_rgb, ex_nrm, ex_dep = extra if extra is not None else (None, None, None)
        return VsxLossDesc(
            gt_rgb=gt.data_ptr(), prior_depth=ptr(pd), prior_depth_valid=ptr(pv),
            prior_normal=ptr(pn), prior_normal_valid=ptr(pnv),
            rgb_scale=1.0 / (B * view.height * view.width * 3),
            depth_weight=(w2 / len(have)) if vi in have else 0.0,
            normal_weight=(wn / len(have_n) / 3.0) if vi in have_n else 0.0,
            sums=sums[vi].data_ptr(), counts=counts[vi].data_ptr(),
            extra_rgb=ptr(ex_rgb), extra_normal=ptr(ex_nrm),
            extra_depth=ptr(ex_dep), live_pairs=live.data_ptr())

    def take_front(vi):
        nonlocal gaussians, isects
        active, dec, P, Bn, ev = fronts.pop(vi)
        hold.append((active, dec, P, Bn))
        with _span(timer, "wait_front"):   # main-stream idle time waiting for the front end
            main.wait_event(ev)
        gaussians += dec.count
        isects += Bn.intersections
        if book is not None:
            book.view_start(vi, active, Bn)
        return active, dec, P, Bn

    def backward(vi, active, dec, P, Bn, R, loss):
        view = views[vi]
        with _span(timer, "raster_bwd"):
            gs = D.raster_backward(P, Bn, view, R, loss=loss, deterministic=cfg.deterministic)
        if book is not None:
            book.view_end(vi)
        # projection + decoder backward of this view run on the tail stream,
        # overlapping the next view's compositor; they are the only writers
        # of the parameter gradients, so one stream keeps them ordered
        if ts is not main:
            ts.wait_stream(main)
        with torch.cuda.stream(ts):
            with _span(timer, "project_bwd"):
                gg = D.project_backward(dec.means, dec.scale, dec.quat, dec.normal, P, gs, view)
                # growth pressure: |dL/dmu| of every gaussian into its anchor
                # (one fused kernel: float64 norms, per-anchor sum and count)
                call("vsx_growth_accumulate", ptr(gg["means"]), ptr(active), int(active.numel()),
                     state.n, ptr(state.grow_sum_flat), ptr(state.grow_cnt_flat), stream())
            with _span(timer, "decode_bwd"):
                decoder_backward_into(params, state.dgrads, active, ds.centers, anchors.emb,
                                      anchors.log_scales, anchors.offsets, view, ds.lod_ref,
                                      ds.max_scale, dec, gg["means"], gg["opacities"],
                                      gg["colors"], gg["scales"], gg["quats"], gg["normals"],
                                      agrads.emb, agrads.log_scales, agrads.offsets)
        hold.append((R, gs, gg))
        if keep is not None:
            keep.append(ViewWork(active, dec, P, Bn, R, gs, gg))

    geo_val, geo_pairs, geo_patches = 0.0, 0, 0
    use_geo = w3 > 0 and B >= 2
    front(0)
    if not use_geo:
        for vi in range(B):
            active, dec, P, Bn = take_front(vi)
            # fused objective (K9 inside K5/K6): loss sums in the forward
            # epilogue, cotangents formed on the fly in the backward
            loss = loss_desc(vi)
            _tr(f"raster{vi}")
            with _span(timer, "raster_fwd"):
                R = D.raster_forward(P, Bn, views[vi], loss=loss, deterministic=cfg.deterministic)
            backward(vi, active, dec, P, Bn, R, loss)
            _tr(f"bwd{vi}_queued")
            # the next view's front end is issued after this view's back end
            # is queued, so it overlaps it on the GPU
            if vi + 1 < B:
                front(vi + 1)
    else:
        # Eq. 10 couples view pairs (losses.py:199-287, trainer.py:309-315):
        # every view is composited first, the NCC cotangents of the source
        # views are formed on the device, then each view runs its backward
        # with them added to the fused objective's cotangents.
        fwd = []
        for vi in range(B):
            active, dec, P, Bn = take_front(vi)
            loss = loss_desc(vi)
            with _span(timer, "raster_fwd"):
                R = D.raster_forward(P, Bn, views[vi], loss=loss, deterministic=cfg.deterministic)
            fwd.append((active, dec, P, Bn, R))
            if vi + 1 < B:
                front(vi + 1)
        from .losses import geo_loss_cotangents
        tg = [SimpleNamespace(rgb=f[4].rgb, normal=f[4].normal, depth=f[4].depth,
                              alpha=f[4].alpha, valid=f[4].valid) for f in fwd]
        with _span(timer, "geo_ncc"):
            g_loss, gstats, cot = geo_loss_cotangents(tg, views, state.rng,
                                                      patch_count=cfg.geo_patches,
                                                      half=cfg.geo_patch_half, upstream=w3)
        geo_val = float(g_loss)
        geo_pairs, geo_patches = gstats.pairs_used, gstats.patches_used
        hold.append(cot)
        for vi in range(B):
            active, dec, P, Bn, R = fwd[vi]
            backward(vi, active, dec, P, Bn, R, loss_desc(vi, cot.get(vi)))
    main.wait_stream(ts)
    # every report scalar in ONE device->host read (the only sync of the
    # step; the non-finite check must precede Adam, trainer.py:317-321)
    hw = torch.tensor([v.height * v.width * 3 for v in views], dtype=torch.float64, device=dev)
    z = torch.zeros((), dtype=torch.float64, device=dev)
    vals = [status[0].double(), (rgb_acc / hw).mean(), z, z, z, tile_max[0].double(),
            live.double()]
    if have:
        cnt = dep_cnt.double()
        terms = torch.where(cnt > 0, dep_sum / cnt.clamp_min(1), torch.zeros_like(cnt))
        vals[2] = terms[have].mean()
        vals[3] = dep_cnt.sum().double()
    if have_n:
        cnt = nrm_cnt.double()
        terms = torch.where(cnt > 0, nrm_sum / (3.0 * cnt.clamp_min(1)), torch.zeros_like(cnt))
        vals[4] = terms[have_n].mean()
    # the non-finite check precedes the update (trainer.py:317-321): Adam is
    # queued before the host read and skips itself on the device when the
    # status bits or the loss are bad, so no host round trip sits in front of
    # it; the host then raises with the parameters untouched
    vt = torch.stack(vals)
    total_dev = vt[1] + w2 * vt[2] + wn * vt[4] + w3 * geo_val
    guard = ((vt[0] != 0) | ~torch.isfinite(total_dev)).to(torch.int32)
    with _span(timer, "adam"):
        state.adam(guard)
    _tr("read")
    host = vt.cpu().numpy()
    _tr("read_done")
    state._inflight = None  # the previous step's buffers are idle now
    st_bits, rgb, depth, supervised, normal = int(host[0]), float(host[1]), float(host[2]), \
        int(host[3]), float(host[4])
    if st_bits:
        D.raise_status(st_bits, "train_step")
    total = rgb + w2 * depth + wn * normal + w3 * geo_val
    if not np.isfinite(total):
        raise NumericalError(f"non-finite loss at step {state.step}: rgb={rgb:.4g} depth={depth:.4g}")
    # per-view buffers stay referenced until the next step's sync point (the
    # GPU may still be running Adam and this step's last kernels)
    state._inflight = hold
    report = StepReport(
        step=state.step, total=total, rgb=rgb, depth=depth, geo=geo_val, w2=w2, w3=w3,
        lr=cosine_lr(state.step, cfg.lr_decoder, cfg), supervised_depth_px=supervised,
        geo_pairs=geo_pairs, geo_patches=geo_patches, gaussians=gaussians,
        transfer_bytes=book.transfer_bytes() if book is not None else 0,
        imbalance=book.imbalance() if book is not None else 1.0,
        max_tile_splats=int(host[5]), seconds=time.perf_counter() - t0,
        intersections=isects, normal=normal, live_pairs=int(host[6]))
    state.step += 1
    return report


class _WorkerBook:
    """The reference's simulated multi-worker bookkeeping of one step
    (``trainer.py:264-268, 276-289, 352-364``), for cfg.workers > 1: the LPT
    patch schedule from the EMA cost model, the bytes moved to each view's
    renderer workers (foreign gaussians x 136 B, ``renderer.py:452-477``) and
    the balance report, whose per-patch seconds are the view's measured
    compositing time (CUDA events, read after the step's one sync) split by
    tile-list length + 1. With one worker both fields are their constants
    (0 bytes, imbalance 1.0), exactly as the reference's."""

    def __init__(self, state, views):
        self.state, self.views = state, views
        W = state.cfg.workers
        self.schedule = schedule_patches(views, W, state.cost_model)
        self.patches_by_view: dict[int, list[int]] = {}
        for j, pr in enumerate(self.schedule.patches):
            self.patches_by_view.setdefault(pr.view_id, []).append(j)
        self.owner = torch.as_tensor(state.assignment.flat_owner().astype(np.int64),
                                     device="cuda")
        self.counts = torch.zeros((len(views), W), dtype=torch.int64, device="cuda")
        self.active_n = [0] * len(views)
        self.tile_counts: list = [None] * len(views)
        self.ev: dict = {}

    def view_start(self, vi, active, Bn) -> None:
        a = active.long()
        self.active_n[vi] = int(a.numel())
        if a.numel():
            self.counts[vi] = torch.bincount(self.owner[a], minlength=self.counts.shape[1])
        self.tile_counts[vi] = Bn.tile_offsets[1:].long() - Bn.tile_offsets[:-1].long()
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev[vi] = [e]

    def view_end(self, vi) -> None:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev[vi].append(e)

    def _renderers(self, v) -> set:
        return {int(self.schedule.workers[j]) for j in self.patches_by_view[v.view_id]}

    def transfer_bytes(self) -> int:
        n = self.state.n
        counts = self.counts.cpu().numpy()
        total = 0
        for vi, v in enumerate(self.views):
            g = self.active_n[vi] * n
            for w in self._renderers(v):
                total += (g - int(counts[vi, w]) * n) * 136   # BYTES_PER_GAUSSIAN
        return int(total)

    def imbalance(self) -> float:
        measured = np.zeros(len(self.schedule.patches))
        for vi, v in enumerate(self.views):
            a, b = self.ev[vi]
            secs = a.elapsed_time(b) / 1e3
            weights = self.tile_counts[vi].cpu().numpy().astype(np.float64) + 1.0
            share = weights / weights.sum()
            for j, sh in zip(self.patches_by_view[v.view_id], share):
                measured[j] = secs * sh
        st = self.state
        return balance_report(st.assignment, self.schedule, measured, epoch=st.step,
                              cost_model=st.cost_model).imbalance


OCTANT_SIGNS = np.array([[sx, sy, sz] for sx in (-1.0, 1.0)
                         for sy in (-1.0, 1.0) for sz in (-1.0, 1.0)])


def grow_anchors(state: TrainState) -> int:
    """Insert finer-level children under voxels with persistent gradient
    strain (``trainer.py:379-454``): a level-k voxel whose mean decoded-position
    gradient norm over the window exceeds ``growth_threshold`` gets its octant
    cells at level k+1 (deduplicated, lattice-sorted) appended, with new
    parameters drawn from ``state.rng`` in the reference's order. The device
    buffers are re-laid out level-major; accumulators reset afterwards."""
    from .scene import quantize
    cfg, scene = state.cfg, state.scene
    old_bases = scene.level_bases.copy()
    gsum = state.grow_sum_flat.cpu().numpy()
    gcnt = state.grow_cnt_flat.cpu().numpy()
    additions: dict = {}
    grown = 0
    for k in range(scene.lod_count - 1):
        lo, hi = int(old_bases[k]), int(old_bases[k + 1])
        cnt, sm = gcnt[lo:hi], gsum[lo:hi]
        if cnt.sum() == 0:
            continue
        mean = np.where(cnt > 0, sm / np.maximum(cnt, 1.0), 0.0)
        parents = np.flatnonzero(mean > cfg.growth_threshold)
        if parents.size == 0:
            continue
        child = scene.levels[k + 1]
        cell = scene.levels[k].cell_size
        cand = (scene.levels[k].centers[parents][:, None, :]
                + OCTANT_SIGNS[None, :, :] * (cell / 4.0)).reshape(-1, 3)
        grid = np.unique(quantize(cand, child.cell_size), axis=0)
        if child.count:
            have = {tuple(g) for g in child.grid}
            fresh = np.array([g for g in grid if tuple(g) not in have],
                             dtype=np.int64).reshape(-1, 3)
        else:
            fresh = grid
        if fresh.size == 0:
            continue
        v_new = len(fresh)
        n = scene.offsets_per_voxel
        emb_dim = child.embeddings.shape[1]
        new_emb = state.rng.uniform(-0.01, 0.01, size=(v_new, emb_dim))
        new_scales = np.full((v_new, 3), child.cell_size)
        new_offsets = state.rng.uniform(-0.5, 0.5, size=(v_new, n, 3))
        child.grid = np.concatenate([child.grid, fresh])
        child.embeddings = np.concatenate([child.embeddings, new_emb])
        child.scales = np.concatenate([child.scales, new_scales])
        child.offsets = np.concatenate([child.offsets, new_offsets])
        child.owner = np.concatenate(
            [child.owner, ((np.arange(v_new) + child.count - v_new) % cfg.workers).astype(np.int32)])
        additions[k + 1] = (new_emb, np.log(new_scales), new_offsets)
        grown += v_new
        state.grow_events.append({"step": state.step, "level": k + 1, "added": v_new,
                                  "parents": int(parents.size)})
    if grown:
        state.assignment = assign_voxels(scene, cfg.workers)
        scene.validate()
        state._insert_anchors(old_bases, additions)
    A = scene.total_voxels
    state.grow_sum_flat = torch.zeros(A, dtype=torch.float64, device="cuda")
    state.grow_cnt_flat = torch.zeros(A, dtype=torch.float64, device="cuda")
    return grown



# ------------------------------------------------------------------ checkpoints

_LEVEL_KEYS = (("embeddings", "emb"), ("log_scales", "log_scales"), ("offsets", "offsets"))


def _moment_slices(state: TrainState):
    """(reference moment name, flat buffer name, row slice) in the reference's
    order: decoder tensors, then per level embeddings / log_scales / offsets."""
    out = [(f"dec/{k}", f"dec/{k}", slice(None)) for k in DecoderParams.param_names(state.n)]
    b = state.scene.level_bases
    for k in range(state.scene.lod_count):
        for key, flat in _LEVEL_KEYS:
            out.append((f"lv{k}/{key}", flat, slice(int(b[k]), int(b[k + 1]))))
    return out


def train_records(state: TrainState) -> dict[str, np.ndarray]:
    """Optimizer / train state as the reference's TRN1 records
    (trainer.py:491-502): step, Adam moments (float64), growth accumulators,
    RNG state."""
    rec = {"meta_i": np.array([state.step, state.cfg.workers], np.int64)}
    f = state.flat
    for name, flat, sl in _moment_slices(state):
        rec[f"adam/{name}/m"] = f.view(f.m, flat)[sl].double().cpu().numpy()
        rec[f"adam/{name}/v"] = f.view(f.v, flat)[sl].double().cpu().numpy()
    gs, gc = state.grow_sum, state.grow_cnt
    for k in sorted(gs):
        rec[f"grow/lv{k}/sum"] = gs[k]
        rec[f"grow/lv{k}/cnt"] = gc[k]
    blob = json.dumps(state.rng.bit_generator.state).encode()
    rec["rng_state"] = np.frombuffer(blob, dtype=np.uint8).copy()
    return rec


def restore_train_records(state: TrainState, rec: dict) -> None:
    """Inverse of train_records (trainer.py:505-516)."""
    state.step = int(rec["meta_i"][0])
    f = state.flat
    with torch.no_grad():
        for name, flat, sl in _moment_slices(state):
            for buf, key in ((f.m, "m"), (f.v, "v")):
                dst = f.view(buf, flat)[sl]
                dst.copy_(torch.as_tensor(rec[f"adam/{name}/{key}"], dtype=torch.float32)
                          .reshape(dst.shape))
        b = state.scene.level_bases
        for k in range(state.scene.lod_count):
            lo, hi = int(b[k]), int(b[k + 1])
            state.grow_sum_flat[lo:hi] = torch.as_tensor(rec[f"grow/lv{k}/sum"])
            state.grow_cnt_flat[lo:hi] = torch.as_tensor(rec[f"grow/lv{k}/cnt"])
    state.rng.bit_generator.state = json.loads(bytes(rec["rng_state"]).decode())


def save_checkpoint(path, state: TrainState):
    """Scene (with the trained anchor parameters), decoder and TRN1 in one
    .vsnap file (trainer.py:519-522), readable by the reference."""
    from .snapshot import save_scene
    state.sync_to_scene()
    return save_scene(path, state.scene, decoder=state.params,
                      extra={"TRN1": train_records(state)})


def load_checkpoint(path, cfg: TrainConfig) -> TrainState:
    """Resume from a .vsnap written by save_checkpoint here or by the
    reference: scene + decoder weights + (when present) optimizer state."""
    from .snapshot import load_scene
    scene, dec, rest = load_scene(path)
    state = TrainState(scene, cfg)
    if dec is not None:
        with torch.no_grad():
            for k, t in state.params.tensors.items():
                t.copy_(dec.tensors[k])
    if "TRN1" in rest:
        restore_train_records(state, rest["TRN1"])
    return state
