"""Device-side pipeline stages over the C ABI (PyTorch = allocator + streams).

Every function here allocates its outputs with torch on the current CUDA
device and launches the corresponding ``vsx_*`` kernels on the current
stream. Nothing here computes on the CPU: without CUDA (or without the
built library) every entry point raises.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream
from .errors import NumericalError
from .geometry import CameraView

EMBED_DIM = 32
HIDDEN = 64
REC_F32 = 16            # sizeof(vsx_splat) / 4
GRAD_F32 = 13           # per-splat gradient record
FWD_WARPS = 4           # warps per CTA of the compositor forward (raster_fwd_pk_kernel<4>)
STATUS_NONPD = 1
STATUS_NONFINITE = 2


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2503_23044_b200 runs on a CUDA (sm_100a) device only; "
                           "there is no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


class Workspace:
    """Grow-only scratch buffer shared by the sort/scan/decode-backward calls."""

    def __init__(self) -> None:
        self.buf: torch.Tensor | None = None

    def get(self, nbytes: int) -> tuple:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device.index != torch.cuda.current_device():
            grow = nbytes if self.buf is None else max(nbytes, int(self.buf.numel() * 1.25))
            self.buf = torch.empty(grow, dtype=torch.uint8, device="cuda")
        return ptr(self.buf), self.buf.numel()


_WORKSPACES: dict[int, Workspace] = {}


def workspace() -> Workspace:
    key = _lib.raw_stream()
    ws = _WORKSPACES.get(key)
    if ws is None:
        ws = _WORKSPACES[key] = Workspace()
    return ws


def _u32(n: int) -> torch.Tensor:
    return torch.empty(max(n, 1), dtype=torch.int32, device="cuda")


# ------------------------------------------------------------------ primitives

SORT_SKIP_CONSTANT = 1
SORT_HIST_IN_WS = 2


def sort_pairs_u64(keys: torch.Tensor, vals: torch.Tensor, n: int, skip_constant: bool = True):
    ko = torch.empty_like(keys)
    vo = torch.empty_like(vals)
    lib = _lib.load()
    wp, wb = workspace().get(lib.vsx_sort_ws_bytes(n))
    call("vsx_sort_pairs_u64", ptr(keys), ptr(vals), ptr(ko), ptr(vo), n, 0, 64,
         SORT_SKIP_CONSTANT if skip_constant else 0, wp, wb, stream())
    return ko, vo


def sort_pairs_u32(keys: torch.Tensor, vals: torch.Tensor, n: int, bits: int,
                   skip_constant: bool = False):
    ko = torch.empty_like(keys)
    vo = torch.empty_like(vals)
    lib = _lib.load()
    wp, wb = workspace().get(lib.vsx_sort_ws_bytes(n))
    call("vsx_sort_pairs_u32", ptr(keys), ptr(vals), ptr(ko), ptr(vo), n, 0, bits,
         SORT_SKIP_CONSTANT if skip_constant else 0, wp, wb, stream())
    return ko, vo


def sort_z_gid(z: torch.Tensor, gid: torch.Tensor, int32: bool = False) -> torch.Tensor:
    """Permutation = lexsort((gid, z)) of positive float64 z (int64 on device,
    or the kernel's int32 with ``int32=True``)."""
    n = int(z.numel())
    order = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    if n == 0:
        return order[:0] if int32 else order[:0].long()
    lib = _lib.load()
    wp, wb = workspace().get(lib.vsx_sort_z_gid_ws_bytes(n))
    z, gid = z.contiguous(), gid.contiguous()   # bound for the kernel's lifetime
    call("vsx_sort_z_gid", ptr(z), ptr(gid), ptr(order), n, wp, wb,
         stream())
    return order[:n] if int32 else order.long()


def exclusive_scan(counts: torch.Tensor, n: int) -> torch.Tensor:
    out = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    wp, wb = workspace().get(lib.vsx_scan_ws_bytes(n))
    call("vsx_scan_u32", ptr(counts), ptr(out), n, wp, wb, stream())
    return out


def select_async(flags: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Ordered indices of non-zero u8 flags, capacity-sized, and the device count."""
    n = int(flags.numel())
    idx = _u32(n)
    cnt = torch.empty(1, dtype=torch.int32, device="cuda")   # written by vsx_select
    lib = _lib.load()
    wp, wb = workspace().get(lib.vsx_sort_ws_bytes(n))
    call("vsx_select", ptr(flags), n, ptr(idx), ptr(cnt), wp, wb, stream())
    return idx, cnt


def select(flags: torch.Tensor) -> torch.Tensor:
    """Ordered indices of non-zero u8 flags (one host sync for the count)."""
    idx, cnt = select_async(flags)
    return idx[: int(cnt.item())]


# ------------------------------------------------------------------ scene

class DeviceScene:
    """Static anchor geometry of a SceneModel in the flat level-major layout.

    centers (A,3) float64 are ``grid * cell`` computed on the host with numpy,
    so they are bit-identical to the reference's ``SceneLevel.centers``.
    """

    def __init__(self, scene) -> None:
        require_cuda()
        self.lod_count = scene.lod_count
        self.lod_ref = float(scene.lod_ref_distance)
        self.lod_bias = int(scene.lod_bias)
        self.n = scene.offsets_per_voxel
        self.base_voxel_size = float(scene.base_voxel_size)
        self.level_bases = scene.level_bases
        self.count = int(self.level_bases[-1])
        self.centers = torch.from_numpy(np.ascontiguousarray(scene.flat_centers())).cuda()
        self.levels = torch.from_numpy(scene.flat_levels()).cuda()
        self.signature = self._signature(scene)

    @staticmethod
    def _signature(scene):
        return (tuple(lv.count for lv in scene.levels), float(scene.lod_ref_distance),
                int(scene.lod_bias), torch.cuda.current_device())

    @property
    def max_scale(self) -> float:
        return 3.0 * self.base_voxel_size

    def cull(self, view: CameraView) -> torch.Tensor:
        mask = torch.empty(max(self.count, 1), dtype=torch.uint8, device="cuda")
        call("vsx_cull", ptr(self.centers), ptr(self.levels), self.count, self.lod_count,
             self.lod_ref, self.lod_bias, view.to_abi(), ptr(mask), stream())
        return mask[: self.count]

    def active(self, view: CameraView) -> torch.Tensor:
        return select(self.cull(view))


def device_scene_for(scene) -> DeviceScene:
    ds = getattr(scene, "_vsx_device", None)
    if ds is None or ds.signature != DeviceScene._signature(scene):
        ds = DeviceScene(scene)
        scene._vsx_device = ds
    return ds


# ------------------------------------------------------------------ decode

@dataclass
class Decoded:
    active: torch.Tensor          # (A') int32 flat anchor ids
    means: torch.Tensor           # (G,3) f64
    opacity: torch.Tensor         # (G,) f32
    color: torch.Tensor           # (G,3)
    scale: torch.Tensor           # (G,3)
    quat: torch.Tensor            # (G,4)
    normal: torch.Tensor          # (G,3)
    cache_h: torch.Tensor | None  # (192, A') f32 feature-major
    cache_o: torch.Tensor | None  # (11n, A')

    @property
    def count(self) -> int:
        return int(self.means.shape[0])


def decode(dec_abi, n: int, active: torch.Tensor, centers: torch.Tensor, emb: torch.Tensor,
           log_scales: torch.Tensor, offsets: torch.Tensor, view: CameraView, lod_ref: float,
           max_scale: float, status: torch.Tensor, keep_cache: bool,
           img: torch.Tensor | None = None) -> Decoded:
    """Decode the active anchors for one view. ``img`` is the decoder weight
    image of the current weights (``decoder_image``), built once per
    optimizer step by the callers that decode several views; None builds it
    here."""
    na = int(active.numel())
    g = na * n
    dev = "cuda"
    means = torch.empty((g, 3), dtype=torch.float64, device=dev)
    opac = torch.empty(g, dtype=torch.float32, device=dev)
    col = torch.empty((g, 3), dtype=torch.float32, device=dev)
    scl = torch.empty((g, 3), dtype=torch.float32, device=dev)
    quat = torch.empty((g, 4), dtype=torch.float32, device=dev)
    nrm = torch.empty((g, 3), dtype=torch.float32, device=dev)
    ld = max((na + 3) // 4 * 4, 4)     # cache_ld() of common.cuh: 16-byte aligned rows
    tc = use_tensor_cores(n)
    ch = torch.empty((192, ld), dtype=torch.float32, device=dev) if keep_cache else None
    # the tensor-core path always stages the raw head outputs in cache_o
    co = torch.empty((11 * n, ld), dtype=torch.float32, device=dev) if keep_cache or tc else None
    if tc:
        if img is None:
            img = decoder_image(dec_abi, n)
        call("vsx_decode_fwd_tc", dec_abi, ptr(img), ptr(active), na, ptr(centers), ptr(emb),
             ptr(log_scales), ptr(offsets), view.to_abi(), lod_ref, max_scale, ptr(means),
             ptr(opac), ptr(col), ptr(scl), ptr(quat), ptr(nrm), ptr(ch), ptr(co), ptr(status),
             stream())
    else:
        call("vsx_decode_fwd", dec_abi, ptr(active), na, ptr(centers), ptr(emb), ptr(log_scales),
             ptr(offsets), view.to_abi(), lod_ref, max_scale, ptr(means), ptr(opac), ptr(col),
             ptr(scl), ptr(quat), ptr(nrm), ptr(ch), ptr(co), ptr(status), stream())
    return Decoded(active, means, opac, col, scl, quat, nrm, ch, co)


def use_tensor_cores(n: int) -> bool:
    """tcgen05 decoder for n <= 13 unless VSX_DECODE_TC=0 (FFMA kernel, for A/B)."""
    import os
    return n <= 13 and os.environ.get("VSX_DECODE_TC", "1") != "0"


def decoder_image(dec_abi, n: int) -> torch.Tensor:
    """3xTF32 hi/lo weight image in the tensor-core shared-memory layout."""
    lib = _lib.load()
    img = torch.empty(int(lib.vsx_decoder_image_floats(n)), dtype=torch.float32, device="cuda")
    call("vsx_decoder_image", dec_abi, ptr(img), stream())
    return img


# ------------------------------------------------------------------ project + sort

@dataclass
class Projected:
    rec: torch.Tensor        # (G',16) f32 view of vsx_splat records, sorted
    radius: torch.Tensor     # (G',) f64 sorted
    zkey_or_thunk: object    # (G',) int64 (float64 z bits) sorted, or a thunk making it
    src: torch.Tensor        # (G',) int32 index into the decode batch
    count: int

    @property
    def zkey(self) -> torch.Tensor:
        """Sorted z keys; gathered on first use (the training step never reads them)."""
        if callable(self.zkey_or_thunk):
            self.zkey_or_thunk = self.zkey_or_thunk()
        return self.zkey_or_thunk

    @property
    def mean2d(self) -> torch.Tensor:
        return self.rec.view(torch.float64)[:, 0:2]

    @property
    def conic(self) -> torch.Tensor:
        return self.rec[:, 4:7]

    @property
    def opacity(self) -> torch.Tensor:
        return self.rec[:, 7]

    @property
    def color(self) -> torch.Tensor:
        return self.rec[:, 8:11]

    @property
    def normal_cam(self) -> torch.Tensor:
        return self.rec[:, 11:14]

    @property
    def plane_d(self) -> torch.Tensor:
        return self.rec[:, 14]


@dataclass
class ProjectLaunch:
    """project_launch() output: unsorted records, the sort order, and the
    device count of kept splats (read by the caller, possibly batched)."""
    rec: torch.Tensor
    key: torch.Tensor
    rad: torch.Tensor
    kept: torch.Tensor
    order: torch.Tensor | None
    g: int


def project_launch(means, opacity, color, scale, quat, normal, view: CameraView,
                   status: torch.Tensor, sort: bool = True) -> ProjectLaunch:
    """K3 projection + (z, batch-order) sort, no host sync. ``sort=False``
    (the sharded step's owners, whose rows the renderer merges in (z, gid)
    order anyway): only the kept splats are compacted, in batch order, by
    one vsx_select pass instead of the radix sort."""
    g = int(means.shape[0])
    rec = torch.empty((max(g, 1), REC_F32), dtype=torch.float32, device="cuda")
    key = torch.empty(max(g, 1), dtype=torch.int64, device="cuda")
    rad = torch.empty(max(g, 1), dtype=torch.float64, device="cuda")
    # sort=False: the kept count comes from the compaction, and the
    # projection's own counter is scratch (not zeroed, never read)
    kept = (torch.zeros if sort or not g else torch.empty)(1, dtype=torch.int32, device="cuda")
    call("vsx_project_fwd", ptr(means), ptr(opacity), ptr(color), ptr(scale), ptr(quat),
         ptr(normal), g, view.to_abi(), ptr(rec), ptr(key), ptr(rad), ptr(kept), ptr(status),
         stream())
    if not g:
        order = None
    elif sort:
        order = sort_splats_z(key[:g], g)
    else:
        # culled splats carry key ~0 (vsx_project_fwd)
        order, kept = select_async((key[:g] != -1).view(torch.uint8))
    return ProjectLaunch(rec, key, rad, kept, order, g)


def project_finish(pl: ProjectLaunch, n_kept: int) -> "Projected":
    if pl.g == 0:
        return Projected(pl.rec[:0], pl.rad[:0], pl.key[:0], pl.kept[:0], 0)
    return gather_projected(pl.rec, pl.key, pl.rad, pl.order, n_kept)


def project(means, opacity, color, scale, quat, normal, view: CameraView,
            status: torch.Tensor) -> Projected:
    """EWA projection + stable (z, batch-order) sort; batch must be gid-ascending."""
    pl = project_launch(means, opacity, color, scale, quat, normal, view, status)
    return project_finish(pl, int(pl.kept.item()) if pl.g else 0)


def sort_splats_z(key: torch.Tensor, g: int) -> torch.Tensor:
    """Stable order by the float64 z bits (proxy sort + exact run fix-up, no sync)."""
    order = torch.empty(max(g, 1), dtype=torch.int32, device="cuda")
    lib = _lib.load()
    wp, wb = workspace().get(lib.vsx_sort_splats_ws_bytes(g))
    call("vsx_sort_splats_z", ptr(key), g, ptr(order), wp, wb, stream())
    return order[:g]


def gather_projected(rec, key, rad, order, n_kept: int) -> "Projected":
    rs = torch.empty((max(n_kept, 1), REC_F32), dtype=torch.float32, device="cuda")
    rr = torch.empty(max(n_kept, 1), dtype=torch.float64, device="cuda")
    call("vsx_gather_splats", ptr(rec), ptr(rad), ptr(order), n_kept, ptr(rs), ptr(rr), stream())
    src = order[:n_kept]
    return Projected(rs[:n_kept], rr[:n_kept], lambda: key[src.long()], src, n_kept)


# ------------------------------------------------------------------ binning

@dataclass
class Bins:
    tile_offsets: torch.Tensor   # (T+1,) int32 (uint32 bits)
    tile_list: torch.Tensor      # (I,) int32 sorted-splat ranks, ascending per tile
    tiles_x: int
    tiles_y: int

    @property
    def intersections(self) -> int:
        return int(self.tile_list.numel())


SEGSORT_CAP = 4096   # vsx_tile_segsort shared-memory capacity


def _binning() -> str:
    """Binning variant: "rowcol" (default: row then column stable counting
    sorts, vsx_bin_plan / vsx_bin_build; images up to 4096 px a side),
    "sort" (emit (tile, rank) pairs + onesweep radix sort; any size) or
    "tiles" (per-tile atomics + per-tile bitonic sort; measured 2.5x slower
    than "sort" on cfg2, kept as an A/B reference)."""
    import os
    return os.environ.get("VSX_BIN", "rowcol")


def _tile_major_binning() -> bool:
    return _binning() == "tiles"


def _bin_rowcol(P: Projected, width: int, height: int, txn: int, tyn: int) -> Bins:
    lib = _lib.load()
    n, T = P.count, txn * tyn
    pb = int(lib.vsx_bin_plan_ws_bytes(n, width, height))
    pw = torch.empty(pb, dtype=torch.uint8, device="cuda")
    tot = torch.empty(2, dtype=torch.int64, device="cuda")
    call("vsx_bin_plan", ptr(P.rec), ptr(P.radius), n, width, height, ptr(pw), pb, ptr(tot),
         stream())
    E, total = (int(x) for x in tot.cpu())   # the front end's one host read
    bb = int(lib.vsx_bin_build_ws_bytes(width, height, E))
    bw = torch.empty(max(bb, 1), dtype=torch.uint8, device="cuda")
    toff = torch.empty(T + 1, dtype=torch.int32, device="cuda")
    lst = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
    call("vsx_bin_build", n, width, height, E, total, ptr(pw), pb, ptr(bw), bb, ptr(toff), ptr(lst),
         stream())
    return Bins(toff, lst[:total], txn, tyn)


def bin_tiles(P: Projected, width: int, height: int) -> Bins:
    txn, tyn = (width + 15) // 16, (height + 15) // 16
    T = txn * tyn
    n = P.count
    if n == 0:
        return Bins(torch.zeros(T + 1, dtype=torch.int32, device="cuda"),
                    torch.empty(0, dtype=torch.int32, device="cuda"), txn, tyn)
    if _binning() == "rowcol" and txn <= 256 and tyn <= 256:
        return _bin_rowcol(P, width, height, txn, tyn)
    if _tile_major_binning():
        # per-tile counts -> CSR offsets -> atomic tile-major emission ->
        # per-tile sort of the ranks (one host read: total and longest list)
        tc = torch.empty(T, dtype=torch.int32, device="cuda")
        call("vsx_bin_count", ptr(P.rec), ptr(P.radius), n, width, height, ptr(None), ptr(tc),
             stream())
        toff = exclusive_scan(tc, T)
        total, longest = (int(x) for x in torch.stack([toff[T].long(), tc.max().long()]).cpu())
        if longest <= SEGSORT_CAP:
            lst = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
            cursor = torch.empty(T, dtype=torch.int32, device="cuda")
            call("vsx_bin_emit_tiles", ptr(P.rec), ptr(P.radius), n, width, height, ptr(toff),
                 ptr(cursor), ptr(lst), stream())
            call("vsx_tile_segsort", ptr(toff), T, ptr(lst), longest, stream())
            return Bins(toff[:T + 1], lst[:total], txn, tyn)
    counts = torch.empty(n, dtype=torch.int32, device="cuda")
    call("vsx_bin_count", ptr(P.rec), ptr(P.radius), n, width, height, ptr(counts), ptr(None),
         stream())
    soff = exclusive_scan(counts, n)
    total = int(soff[n].item())
    if total == 0:
        return Bins(torch.zeros(T + 1, dtype=torch.int32, device="cuda"),
                    torch.empty(0, dtype=torch.int32, device="cuda"), txn, tyn)
    tiles = torch.empty(total, dtype=torch.int32, device="cuda")
    ranks = torch.empty(total, dtype=torch.int32, device="cuda")
    bits = max(1, math.ceil(math.log2(T))) if T > 1 else 1
    lib = _lib.load()
    if T <= 65536:
        # the emission builds the sort's digit histograms on the fly
        wp, wb = workspace().get(lib.vsx_sort_ws_bytes(total))
        hist = wp + int(lib.vsx_sort_hist_offset(total))
        call("vsx_bin_emit_hist", ptr(P.rec), ptr(P.radius), n, width, height, ptr(soff),
             ptr(tiles), ptr(ranks), hist, stream())
        skeys = torch.empty_like(tiles)
        lst = torch.empty_like(ranks)
        call("vsx_sort_pairs_u32", ptr(tiles), ptr(ranks), ptr(skeys), ptr(lst), total, 0, bits,
             SORT_HIST_IN_WS, wp, wb, stream())
    else:
        call("vsx_bin_emit", ptr(P.rec), ptr(P.radius), n, width, height, ptr(soff),
             ptr(tiles), ptr(ranks), stream())
        skeys, lst = sort_pairs_u32(tiles, ranks, total, bits)
    toff = torch.empty(T + 1, dtype=torch.int32, device="cuda")
    call("vsx_tile_ranges", ptr(skeys), total, T, ptr(toff), stream())
    return Bins(toff, lst, txn, tyn)


# ------------------------------------------------------------------ raster

@dataclass
class Raster:
    rgb: torch.Tensor
    alpha: torch.Tensor
    depth: torch.Tensor
    normal: torch.Tensor
    raw_normal: torch.Tensor
    valid: torch.Tensor          # uint8
    t_final: torch.Tensor
    n_contrib: torch.Tensor


def raster_forward(P: Projected, B: Bins, view: CameraView, loss=None,
                   deterministic: bool = False) -> Raster:
    """K5; with a VsxLossDesc the fused objective's sums/counts are accumulated
    too (deterministic: per-(tile, warp) partial sums reduced in a fixed order
    instead of float atomics)."""
    H, W = view.height, view.width
    dev = "cuda"
    rgb = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    alpha = torch.empty((H, W), dtype=torch.float32, device=dev)
    depth = torch.empty((H, W), dtype=torch.float32, device=dev)
    normal = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    raw = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    valid = torch.empty((H, W), dtype=torch.uint8, device=dev)
    tfin = torch.empty((H, W), dtype=torch.float32, device=dev)
    nc = torch.empty((H, W), dtype=torch.int32, device=dev)
    if loss is None:
        call("vsx_raster_fwd", ptr(P.rec), ptr(B.tile_offsets), ptr(B.tile_list), view.to_abi(),
             ptr(rgb), ptr(alpha), ptr(depth), ptr(normal), ptr(raw), ptr(valid), ptr(tfin),
             ptr(nc), stream())
    else:
        part = None
        if deterministic:
            slots = B.tiles_x * B.tiles_y * FWD_WARPS
            part = torch.zeros((slots, 3), dtype=torch.float64, device=dev)
            loss.sum_partials = part.data_ptr()
        call("vsx_raster_fwd_loss", ptr(P.rec), ptr(B.tile_offsets), ptr(B.tile_list),
             view.to_abi(), ptr(rgb), ptr(alpha), ptr(depth), ptr(normal), ptr(raw), ptr(valid),
             ptr(tfin), ptr(nc), loss, stream())
        if part is not None:
            loss.sum_partials = None
            call("vsx_reduce_partials", ptr(part), int(part.shape[0]), ctypes.c_void_p(loss.sums),
                 stream())
    return Raster(rgb, alpha, depth, normal, raw, valid, tfin, nc)


def _tile_order_enabled() -> bool:
    import os
    return os.environ.get("VSX_TILE_ORDER", "0") == "1"


def raster_backward(P: Projected, B: Bins, view: CameraView, R: Raster, g_rgb=None, g_alpha=None,
                    g_depth=None, g_normal=None, g_raw=None, out: torch.Tensor | None = None,
                    loss=None, deterministic: bool = False):
    """K6 from explicit pixel cotangents, or (loss=VsxLossDesc) from the fused
    objective (deterministic: per-intersection gradient rows reduced per
    splat in tile order instead of float atomics)."""
    grad = out if out is not None else torch.zeros((max(P.count, 1), GRAD_F32),
                                                   dtype=torch.float32, device="cuda")
    if loss is not None:
        order = None
        if _tile_order_enabled() and B.tile_list.numel():
            # heaviest tiles first: the long tiles start in the first wave
            # instead of forming the kernel's tail
            lens = B.tile_offsets[1:] - B.tile_offsets[:-1]
            order = torch.argsort(lens, descending=True).to(torch.int32)
            loss.tile_order = order.data_ptr()
        rows = live = None
        if deterministic and B.intersections:
            rows = torch.empty((B.intersections, GRAD_F32), dtype=torch.float32, device="cuda")
            # zeros: a band launch leaves the other tiles' live counts unset
            live = torch.zeros(B.tiles_x * B.tiles_y, dtype=torch.int32, device="cuda")
            loss.isect_grad, loss.tile_live = rows.data_ptr(), live.data_ptr()
        call("vsx_raster_bwd_loss", ptr(P.rec), ptr(B.tile_offsets), ptr(B.tile_list),
             view.to_abi(), ptr(R.rgb), ptr(R.alpha), ptr(R.depth), ptr(R.normal),
             ptr(R.raw_normal), ptr(R.t_final), ptr(R.n_contrib), loss, ptr(grad), stream())
        if rows is not None:
            loss.isect_grad = loss.tile_live = None
            call("vsx_raster_grad_reduce", ptr(P.rec), ptr(P.radius), P.count, view.width,
                 view.height, ptr(B.tile_offsets), ptr(B.tile_list), ptr(live), ptr(rows),
                 ptr(grad), stream())
        return grad[: P.count]
    call("vsx_raster_bwd", ptr(P.rec), ptr(B.tile_offsets), ptr(B.tile_list), view.to_abi(),
         ptr(R.rgb), ptr(R.alpha), ptr(R.depth), ptr(R.raw_normal), ptr(R.t_final),
         ptr(R.n_contrib), ptr(g_rgb), ptr(g_alpha), ptr(g_depth), ptr(g_normal), ptr(g_raw),
         ptr(grad), stream())
    return grad[: P.count]


def project_backward(means, scale, quat, normal, P: Projected, grad_splat: torch.Tensor,
                     view: CameraView):
    g = int(means.shape[0])
    dev = "cuda"
    # batch-order kernel: every row written (zeros for culled gaussians)
    gm = torch.empty((g, 3), dtype=torch.float32, device=dev)
    go = torch.empty(g, dtype=torch.float32, device=dev)
    gc = torch.empty((g, 3), dtype=torch.float32, device=dev)
    gs = torch.empty((g, 3), dtype=torch.float32, device=dev)
    gq = torch.empty((g, 4), dtype=torch.float32, device=dev)
    gn = torch.empty((g, 3), dtype=torch.float32, device=dev)
    inv = torch.empty(max(g, 1), dtype=torch.int32, device=dev)
    call("vsx_project_bwd_batch", ptr(means), ptr(scale), ptr(quat), ptr(normal), ptr(P.rec),
         ptr(grad_splat), P.count, g, view.to_abi(), ptr(gm), ptr(go), ptr(gc), ptr(gs),
         ptr(gq), ptr(gn), ptr(P.src if P.src.dtype == torch.int32 else None), ptr(inv), stream())
    return {"means": gm, "opacities": go, "colors": gc, "scales": gs, "quats": gq, "normals": gn}


def check_status(status: torch.Tensor, what: str) -> None:
    s = int(status.item())
    if s & STATUS_NONPD:
        raise NumericalError(f"{what}: non positive definite 2d covariance")
    if s & STATUS_NONFINITE:
        raise NumericalError(f"{what}: non-finite decoder output")


def raise_status(bits: int, what: str) -> None:
    """check_status on an already-read status word."""
    if bits & STATUS_NONPD:
        raise NumericalError(f"{what}: non positive definite 2d covariance")
    if bits & STATUS_NONFINITE:
        raise NumericalError(f"{what}: non-finite decoder output")
