"""Multi-GPU training step: anchors sharded by the paper's Eq. 3, splats exchanged.

One process per GPU. Each rank owns the anchors with ``i mod M == rank`` per
level (``partition.assign_voxels``, reference ``partition.py:43-52``) and, for
EVERY view of the batch, culls/decodes/projects only those anchors. View ``v``
is rendered by rank ``v mod M``. Per step:

* **C1 forward** (``exchange_splats``): an all-to-all of the projected splat
  payloads (64-byte record + float64 z, radius and int64 gid per splat) from
  the owners to each view's renderer. The reference only accounts these bytes
  (``renderer.py:452-477``); here they really move (NCCL over NVLink).
* The renderer merges the segments, restores the exact reference order
  ``lexsort((gid, z))`` (stable z sort + gid tie fix), bins, composites, and
  back-propagates the fused loss to per-splat gradients (13 floats).
* **C1 backward** (``return_grads``): the reverse all-to-all sends each owner
  the gradients of its own splats, which then runs projection and decode
  backward locally. Anchor gradients and their Adam stay owner-local.
* **C2**: an all-reduce SUM of the decoder gradient (the reference sums over
  all views and anchors in one autograd call, ``trainer.py:330``), then the
  replicated decoder Adam keeps every replica bit-identical.

The compute is behind a small backend interface so the routing is testable
without GPUs: ``CudaShardBackend`` (below) drives the sm_100a kernels;
``oracle.shard.OracleShardBackend`` (test infrastructure) drives the float64
oracle, and ``tests/test_dist_gloo.py`` checks a 2-rank gloo run against the
single-process oracle step.
"""

from __future__ import annotations

from ctypes import c_void_p
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import InvalidInput, ProtocolError


@dataclass
class SplatPayload:
    """Projected splats of one (rank, view): rows aligned across the tensors."""

    rec: torch.Tensor     # (n, R) record words (R = 16 float32 on CUDA)
    z: torch.Tensor       # (n,) float64 camera depth (sort key)
    radius: torch.Tensor  # (n,) float64 3-sigma radius (binning)
    gid: torch.Tensor     # (n,) int64 global gaussian id (tie break)

    @property
    def count(self) -> int:
        return int(self.z.shape[0])

    @staticmethod
    def cat(parts: list["SplatPayload"], like: "SplatPayload") -> "SplatPayload":
        if not parts:
            return SplatPayload(like.rec[:0], like.z[:0], like.radius[:0], like.gid[:0])
        return SplatPayload(torch.cat([p.rec for p in parts]), torch.cat([p.z for p in parts]),
                            torch.cat([p.radius for p in parts]),
                            torch.cat([p.gid for p in parts]))


def renderer_of(view_index: int, world: int) -> int:
    return view_index % world


ROW_BYTES = 96   # VSX_SPLAT_ROW_BYTES: record | z | radius | gid | pad


@dataclass
class PackedPayload:
    """A renderer's received rows of one view, left in the all-to-all buffer:
    row i of the view is ``rows[rowmap[i]]`` (``rowmap`` None: row ``base + i``);
    z and gid are extracted for the (z, gid) merge sort."""

    buf: torch.Tensor            # (N, ROW_BYTES) uint8 receive buffer
    base: int                    # first row of the view when rowmap is None
    rowmap: torch.Tensor | None  # (n,) int32 rows of buf, source-rank order
    z: torch.Tensor              # (n,) float64
    gid: torch.Tensor            # (n,) int64

    @property
    def count(self) -> int:
        return int(self.z.shape[0])

    def rows_ptr(self) -> int:
        return self.buf.data_ptr() + (self.base if self.rowmap is None else 0) * ROW_BYTES


def _cuda_rows(p: SplatPayload) -> bool:
    return (p.rec.is_cuda and p.rec.dtype == torch.float32 and p.rec.dim() == 2
            and p.rec.shape[1] == 16)


def _pack_rows(parts: list[SplatPayload], total: int, device) -> torch.Tensor:
    """The send buffer of the CUDA path: every part's rows packed in order by
    vsx_pack_splat_rows (one pass, no intermediate concatenation)."""
    from ._lib import call, ptr, stream
    buf = torch.empty((max(total, 1), ROW_BYTES), dtype=torch.uint8, device=device)
    off = 0
    for p in parts:
        n = p.count
        if n:
            rec, z = p.rec.contiguous(), p.z.contiguous()
            rad, gid = p.radius.contiguous(), p.gid.contiguous()
            call("vsx_pack_splat_rows", ptr(rec), ptr(z), ptr(rad), ptr(gid), n,
                 c_void_p(buf.data_ptr() + off * ROW_BYTES), stream())
        off += n
    return buf[:total]


def _fields(p: SplatPayload):
    return (p.rec, p.z, p.radius, p.gid)


def _pack(p: SplatPayload) -> torch.Tensor:
    """Rows of all four payload tensors side by side as bytes, (n, row_bytes) u8."""
    n = p.count
    return torch.cat([t.contiguous().view(torch.uint8).reshape(n, -1) for t in _fields(p)], 1)


def _unpack(buf: torch.Tensor, like: SplatPayload) -> SplatPayload:
    n = int(buf.shape[0])
    out, col = [], 0
    for t in _fields(like):
        width = t.element_size() * int(np.prod(t.shape[1:], dtype=np.int64))
        part = buf[:, col:col + width].contiguous().view(t.dtype)
        out.append(part.reshape((n,) + tuple(t.shape[1:])))
        col += width
    return SplatPayload(*out)


def _a2a(x: torch.Tensor, in_splits: list[int], out_splits: list[int], group=None):
    out = torch.empty((sum(out_splits),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    dist.all_to_all_single(out, x.contiguous(), out_splits, in_splits, group=group)
    return out


@dataclass
class ExchangePlan:
    """Per-(source rank, view) row counts of one step's C1 exchange."""

    counts: np.ndarray        # (world, B): rows rank q contributes to view v
    rank: int
    world: int
    renderers: np.ndarray | None = None   # (B,) renderer rank of each view

    def __post_init__(self) -> None:
        B = self.counts.shape[1]
        if self.renderers is None:
            self.renderers = np.array([renderer_of(v, self.world) for v in range(B)])
        self.renderers = np.asarray(self.renderers, dtype=np.int64)
        if self.renderers.shape != (B,) or np.any((self.renderers < 0) |
                                                   (self.renderers >= self.world)):
            raise ProtocolError("renderer ranks must be one valid rank per view")

    def views_of(self, r: int) -> list[int]:
        return [v for v in range(self.counts.shape[1]) if int(self.renderers[v]) == r]

    def send_splits(self) -> list[int]:
        return [int(self.counts[self.rank, self.views_of(r)].sum()) for r in range(self.world)]

    def recv_splits(self) -> list[int]:
        mine = self.views_of(self.rank)
        return [int(self.counts[q, mine].sum()) for q in range(self.world)]


def exchange_splats(payloads: list[SplatPayload], rank: int, world: int, group=None,
                    renderers=None):
    """C1 forward: route every view's payload rows to its renderer rank.

    Returns (plan, merged) where merged[v] (for the views this rank renders)
    is the concatenation of all ranks' rows in source-rank order, plus the
    per-source row offsets inside it.
    """
    B = len(payloads)
    dev = payloads[0].z.device
    mine_counts = torch.tensor([p.count for p in payloads], dtype=torch.int64, device=dev)
    gathered = [torch.zeros_like(mine_counts) for _ in range(world)]
    dist.all_gather(gathered, mine_counts, group=group)
    plan = ExchangePlan(torch.stack(gathered).cpu().numpy(), rank, world, renderers)
    send_parts = [payloads[v] for r in range(world) for v in plan.views_of(r)]
    ins, outs = plan.send_splits(), plan.recv_splits()
    mine = plan.views_of(rank)
    if _cuda_rows(payloads[0]):
        return plan, _exchange_rows(plan, send_parts, ins, outs, mine, dev, group)
    send = SplatPayload.cat(send_parts, payloads[0])
    # ONE all-to-all of packed rows (record | z | radius | gid bytes)
    recv = _unpack(_a2a(_pack(send), ins, outs, group), payloads[0])
    # split the received block per (source, view) and regroup per view
    merged: dict[int, tuple[SplatPayload, list[int]]] = {}
    pieces: dict[int, list[SplatPayload]] = {v: [] for v in mine}
    off = 0
    for q in range(world):
        for v in mine:
            c = int(plan.counts[q, v])
            pieces[v].append(SplatPayload(recv.rec[off:off + c], recv.z[off:off + c],
                                          recv.radius[off:off + c], recv.gid[off:off + c]))
            off += c
    for v in mine:
        seg = [0] + list(np.cumsum([int(plan.counts[q, v]) for q in range(world)]))
        merged[v] = (SplatPayload.cat(pieces[v], payloads[0]), seg)
    return plan, merged


def _exchange_rows(plan: ExchangePlan, send_parts, ins, outs, mine, dev, group):
    """C1 forward of the CUDA path: one all-to-all of 96-byte rows packed by
    vsx_pack_splat_rows; each view's rows stay in the receive buffer (a row
    map when they come from several sources) and only the sort keys are
    extracted (vsx_splat_rows_keys)."""
    from ._lib import call, ptr, stream
    world = plan.world
    recv = _a2a(_pack_rows(send_parts, sum(ins), dev), ins, outs, group)
    starts: dict[int, list[tuple[int, int]]] = {v: [] for v in mine}
    off = 0
    for q in range(world):
        for v in mine:
            c = int(plan.counts[q, v])
            starts[v].append((off, c))
            off += c
    merged = {}
    for v in mine:
        blocks = [(o, c) for o, c in starts[v] if c]
        n = sum(c for _, c in blocks)
        rowmap, base = None, (blocks[0][0] if blocks else 0)
        if len(blocks) > 1:
            rowmap = torch.cat([torch.arange(o, o + c, dtype=torch.int32, device=dev)
                                for o, c in blocks])
        z = torch.empty(max(n, 1), dtype=torch.float64, device=dev)[:n]
        gid = torch.empty(max(n, 1), dtype=torch.int64, device=dev)[:n]
        pl = PackedPayload(recv, base, rowmap, z, gid)
        if n:
            call("vsx_splat_rows_keys", c_void_p(pl.rows_ptr()), ptr(rowmap), n, ptr(z),
                 ptr(gid), stream())
        seg = [0] + list(np.cumsum([int(plan.counts[q, v]) for q in range(world)]))
        merged[v] = (pl, seg)
    return merged


def return_grads(plan: ExchangePlan, grads: dict[int, torch.Tensor], like: torch.Tensor,
                 group=None) -> list[torch.Tensor]:
    """C1 backward: send each source its rows' gradients; returns per-view grads
    aligned with this rank's own payloads."""
    rank, world = plan.rank, plan.world
    mine = plan.views_of(rank)
    blocks = []
    for q in range(world):
        for v in mine:
            g = grads[v]
            seg = np.concatenate([[0], np.cumsum(plan.counts[:, v])])
            blocks.append(g[int(seg[q]):int(seg[q + 1])])
    send = torch.cat(blocks) if blocks else like[:0]
    recv = _a2a(send, plan.recv_splits(), plan.send_splits(), group)
    out: list[torch.Tensor | None] = [None] * plan.counts.shape[1]
    off = 0
    for r in range(world):
        for v in plan.views_of(r):
            c = int(plan.counts[rank, v])
            out[v] = recv[off:off + c]
            off += c
    return out


def _unsort_rows(gs: torch.Tensor, order: torch.Tensor) -> torch.Tensor:
    """merged[order[i]] = gs[i]: sorted-splat gradient rows back to the
    received row order (vsx_scatter_rows_f32)."""
    from ._lib import call, ptr, stream
    merged = torch.empty_like(gs)
    n = int(order.numel())
    if n:
        o32 = order if order.dtype == torch.int32 else order.int()
        g = gs.contiguous()
        call("vsx_scatter_rows_f32", ptr(g), ptr(o32), n, int(gs.shape[1]), ptr(merged), stream())
    return merged


class _StagedView:
    """Indexable view of one input kind of an _InputStager (0 = image,
    1 = depth prior, 2 = normal prior); indexing waits for the view's copy."""

    def __init__(self, stager, kind):
        self.stager, self.kind = stager, kind

    def __getitem__(self, v):
        gt, pd, pv, pn, pnv = self.stager.get(v)
        if self.kind == 0:
            return gt
        if self.kind == 1:
            return None if pd is None else (pd, pv)
        return None if pn is None else (pn, pnv)


def _StagedInputs(stager, B):
    return _StagedView(stager, 0), _StagedView(stager, 1), _StagedView(stager, 2)


def sharded_train_step(backend, views, images, priors=None, normal_priors=None, group=None,
                       scheduler=None):
    """One sharded step; returns the global loss terms (same on every rank).

    With a ``partition.ViewScheduler`` the renderer rank of every view comes
    from LPT over the EMA of each view's measured render seconds (the
    reference's patch scheduler, ``partition.py:84-207``, applied to whole
    views); the per-view times are summed across ranks so every rank folds
    identical measurements into its model and picks the same assignment.
    """
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    B = len(views)
    w2, w3, wn = backend.schedule()
    use_geo = w3 > 0 and B >= 2
    if use_geo and not hasattr(backend, "band_forward"):
        # Eq. 10 couples views that different ranks render (losses.py:196-287)
        raise InvalidInput("the Eq. 10 multi-view NCC term (w3 > 0) needs the two-phase "
                           "sharded step (CudaShardBackend)")
    # the depth / normal terms average over the views that carry a prior
    # (trainer.py:296-306, losses.py:84), a global property of the batch
    have = [v for v in range(B) if w2 > 0 and priors is not None and priors[v] is not None]
    have_n = [v for v in range(B)
              if wn > 0 and normal_priors is not None and normal_priors[v] is not None]
    banded = B < world or use_geo
    if banded:
        # fewer views than ranks: every view is split into tile-row bands, one
        # work item each, dealt round-robin over the ranks (SURVEY §8(e) step
        # 2: "tile bands of a view when B < M"; the reference's patch work
        # items, partition.py:71-81)
        if not hasattr(backend, "band_forward"):
            raise InvalidInput("a batch with fewer views than ranks needs tile bands "
                               "(CudaShardBackend)")
        if B < world:
            S = -(-world // B)
            bands = {v: backend.band_rows(views[v], S) for v in range(B)}
            items = [(v, b) for v in range(B) for b in range(len(bands[v]))]
            item_rend = np.arange(len(items), dtype=np.int64) % world
        else:
            # whole views (one band each) on their round-robin renderers: the
            # two-phase path only for the NCC term's exchange of renders
            bands = {v: [(0, (views[v].height + 15) // 16)] for v in range(B)}
            items = [(v, 0) for v in range(B)]
            item_rend = np.asarray([renderer_of(v, world) for v in range(B)], dtype=np.int64)
        renderers = np.asarray([renderer_of(v, world) for v in range(B)], dtype=np.int64)
        mine = {v for (v, _), r in zip(items, item_rend) if int(r) == rank}
    else:
        renderers = scheduler.assign(views, world) if scheduler is not None else None
        renderers = np.asarray(renderers if renderers is not None
                               else [renderer_of(v, world) for v in range(B)], dtype=np.int64)
        mine = {v for v in range(B) if int(renderers[v]) == rank}
    backend.begin_step(views, have, have_n)
    from .trainer import _InputStager, _pipeline_enabled, _prior_arrays
    if hasattr(backend, "prepare"):
        # the targets / priors of the views this rank renders go to the
        # device up front on the copy stream (non-blocking from pinned host
        # memory), each view's compositor waiting only for its own inputs
        dpri = None if priors is None else [_prior_arrays(p) for p in priors]
        stager = _InputStager(views, images, dpri, set(have), normal_priors, set(have_n),
                              only=mine)
        images, priors, normal_priors = _StagedInputs(stager, B)
    if banded:
        timers = _banded_views(backend, views, images, priors, normal_priors, group, rank, world,
                               bands, items, item_rend, use_geo)
    elif hasattr(backend, "prepare") and _pipeline_enabled():
        timers = _pipelined_views(backend, views, images, priors, normal_priors, group,
                                  renderers, rank, world)
    else:
        payloads = [backend.forward_shard(v, views[v]) for v in range(B)]
        plan, merged = exchange_splats(payloads, rank, world, group, renderers)
        grads, timers = {}, {}
        for v, (payload, seg) in merged.items():
            t0 = _Stopwatch(payload.z.device)
            grads[v] = backend.render(v, views[v], payload, images[v],
                                      None if priors is None else priors[v],
                                      None if normal_priors is None else normal_priors[v])
            timers[v] = t0.stop()
        back = return_grads(plan, grads, backend.grad_like(), group)
        for v in range(B):
            backend.backward_shard(v, views[v], back[v])
    _c2_sum(backend.decoder_grad(), group, ordered=bool(getattr(backend, "deterministic", False)))
    losses = backend.loss_terms()              # (B, 5): rgb, depth, normal sums; counts
    dist.all_reduce(losses, op=dist.ReduceOp.SUM, group=group)
    report = backend.finish_step(losses)
    check_replicas(backend.decoder_checksum(), group)
    secs = torch.zeros(B, dtype=torch.float64)
    for v, t in timers.items():
        secs[v] = t.seconds()
    if dist.get_backend(group) == "nccl":
        secs = secs.cuda()
    dist.all_reduce(secs, op=dist.ReduceOp.SUM, group=group)
    secs = secs.cpu().numpy()
    per_rank = np.bincount(renderers, weights=secs, minlength=world)
    if isinstance(report, dict):
        report["render_seconds"] = per_rank.tolist()
        report["imbalance"] = float(per_rank.max() / per_rank.mean()) if per_rank.sum() > 0 \
            else 1.0
    if scheduler is not None and not banded:
        scheduler.update(views, secs)
    return report


def _banded_views(backend, views, images, priors, normal_priors, group, rank, world, bands,
                  items, item_rend, use_geo=False) -> dict:
    """The sharded step with views split into tile-row bands (B < M).

    Owners run their shard's front end once per view; C1 sends every band's
    renderer the rows whose tile rectangle reaches its rows (a splat spanning
    two bands goes to both). Each renderer merges, bins over the whole view
    (the band's tile lists are the full view's) and composites only its rows.
    The depth / normal terms are means over a view's valid pixels, so every
    band's forward runs first, the per-band counts are summed per view over
    the ranks, and the backward normalises by the view's total. The reverse
    C1 returns each band's gradients; the owner adds a splat's bands
    together (distinct indices per band) before its projection / decoder
    backward.
    """
    B = len(views)
    payloads = [backend.forward_shard(v, views[v]) for v in range(B)]
    item_payloads, index = [], []
    for v, b in items:
        sub, idx = backend.band_payload(payloads[v], views[v], bands[v][b])
        item_payloads.append(sub)
        index.append(idx)
    plan, merged = exchange_splats(item_payloads, rank, world, group, item_rend)
    backend.begin_bands(len(items))
    for it, (payload, _seg) in merged.items():
        v, b = items[it]
        work = backend.prepare(it, views[v], payload)
        backend.band_forward(it, v, views[v], work, images[v],
                             None if priors is None else priors[v],
                             None if normal_priors is None else normal_priors[v], bands[v][b])
    geo = None
    if use_geo:
        geo = _exchange_renders_and_geo(backend, views, items, item_rend, bands, rank, group)
        backend.geo = geo
    local = backend.icounts.clone()
    tot = local.clone()
    dist.all_reduce(tot, op=dist.ReduceOp.SUM, group=group)
    item_view = torch.tensor([v for v, _ in items], dtype=torch.int64, device=tot.device)
    vt = torch.zeros((B, 2), dtype=tot.dtype, device=tot.device).index_add_(0, item_view, tot)
    for it in merged:
        backend.icounts[it].copy_(vt[items[it][0]])
    grads = {it: backend.band_backward(it, None if geo is None else geo[2].get(items[it][0]))
             for it in merged}
    like = backend.grad_like()
    back = return_grads(plan, grads, like, group)
    for v in range(B):
        g = torch.zeros((payloads[v].count, like.shape[1]), dtype=like.dtype, device=like.device)
        for it, (vv, _b) in enumerate(items):
            if vv == v and back[it] is not None and back[it].numel():
                g.index_add_(0, index[it], back[it])
        backend.backward_shard(v, views[v], g)
    # this rank's share of each view's loss sums / counts (summed over ranks
    # with the other loss terms)
    backend.sums.index_add_(0, item_view, backend.isums)
    backend.counts.index_add_(0, item_view, local)
    return {}


def _exchange_renders_and_geo(backend, views, items, item_rend, bands, rank, group):
    """All views' renders on every rank (each rank contributes the rows it
    composited, one all-reduce SUM), then the Eq. 10 value and cotangents,
    identical on every rank. Returns (value, stats, cot)."""
    from types import SimpleNamespace
    from .losses import geo_loss_cotangents
    dev = "cuda"
    full = []
    for v, view in enumerate(views):
        H, W = view.height, view.width
        full.append(torch.zeros((H, W, 9), dtype=torch.float32, device=dev))
    for it, (_work, view, _loss, _keep, R) in backend.pending.items():
        v, b = items[it]
        r0, nr = bands[v][b]
        y0, y1 = 16 * r0, min(view.height, 16 * (r0 + nr))
        f = full[v]
        f[y0:y1, :, 0:3] = R.rgb[y0:y1]
        f[y0:y1, :, 3:6] = R.normal[y0:y1]
        f[y0:y1, :, 6] = R.depth[y0:y1]
        f[y0:y1, :, 7] = R.alpha[y0:y1]
        f[y0:y1, :, 8] = R.valid[y0:y1].float()
    flat = torch.cat([f.reshape(-1) for f in full])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    tg, off = [], 0
    for v, view in enumerate(views):
        n = view.height * view.width * 9
        f = flat[off:off + n].view(view.height, view.width, 9)
        off += n
        tg.append(SimpleNamespace(rgb=f[..., 0:3].contiguous(), normal=f[..., 3:6].contiguous(),
                                  depth=f[..., 6].contiguous(), alpha=f[..., 7].contiguous(),
                                  valid=f[..., 8] > 0.5))
    st = backend.state
    _w2, w3, _wn = backend.schedule()
    g_loss, gstats, cot = geo_loss_cotangents(tg, views, st.rng, patch_count=st.cfg.geo_patches,
                                              half=st.cfg.geo_patch_half, upstream=w3)
    return float(g_loss), gstats, cot


def _c2_sum(t: torch.Tensor, group, ordered: bool) -> None:
    """C2: the decoder gradient summed over the ranks, in place. ``ordered``
    (deterministic mode): an all-gather and a sum in rank
    order, so the result does not depend on the collective's reduction
    order; otherwise one all-reduce SUM."""
    if not ordered:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t.contiguous(), group=group)
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    t.copy_(acc)


def _shard_groups() -> int:
    import os
    return max(1, int(os.environ.get("VSX_SHARD_GROUPS", "4")))


def _pipelined_views(backend, views, images, priors, normal_priors, group, renderers, rank,
                     world) -> dict:
    """The sharded step in K view groups, software-pipelined over three streams.

    Group k's C1 exchange, compositing and reverse C1 run on the main stream;
    meanwhile the high-priority front stream runs the (z, gid) merge + binning
    of the next composited view and the shard forwards (cull, decode,
    project) of group k+1, and the tail stream runs the shard backwards
    (projection + decoder backward) of group k-1. Every rank issues the same
    collectives in the same order (exchange(g0), return(g0), exchange(g1),
    ...); the side work is rank-local, so ranks may interleave it
    differently. Buffers stay referenced until the step's host sync.
    """
    from .trainer import _front_stream, _side_stream, _tail_stream, _tr
    B = len(views)
    K = min(_shard_groups(), B)
    groups = [list(range(k * B // K, (k + 1) * B // K)) for k in range(K)]
    groups = [g for g in groups if g]
    main = torch.cuda.current_stream()
    # prep (merge + bin) and the shard forwards both read counts back to the
    # host; on separate streams neither read waits behind the other's kernels
    fs, ts = _front_stream(), _tail_stream()
    ss = _side_stream("shard_fwd", priority=-1)
    for st in (fs, ts, ss):
        st.wait_stream(main)
    payloads, hold, timers = {}, [], {}

    def fwd_stepper(g):
        """One stage of the batched shard forward of group g per call."""
        gen = backend.forward_shards(g, views)

        def step():
            with torch.cuda.stream(ss):
                try:
                    next(gen)
                except StopIteration as e:
                    payloads.update(e.value)
        return step

    def bwd(v, g):
        with torch.cuda.stream(ts):
            backend.backward_shard(v, views[v], g)

    _tr("step")
    first = fwd_stepper(groups[0])
    for _ in range(3):
        first()
    _tr("fwd_g0")
    def exchange(k):
        # issued on the shard-forward stream: the NCCL ops wait for that
        # stream's forwards only, not for the compositor work queued on main,
        # and the count read-back syncs that stream only. It is issued before
        # the previous group's reverse exchange, so it does not queue behind it
        # on the communicator either.
        gk = groups[k]
        _tr(f"x{k}")
        with torch.cuda.stream(ss):
            plan, merged = exchange_splats([payloads[v] for v in gk], rank, world, group,
                                           renderers[gk])
        _tr(f"x{k}_done")
        hold.append((plan, merged, [payloads[v] for v in gk]))
        return plan, merged

    pending_bwd: list = []
    nxt = exchange(0)
    for k, gk in enumerate(groups):
        plan, merged = nxt
        fs.wait_stream(ss)            # the merge reads the received rows
        items = list(merged.items())  # (local index, (payload, seg))
        # the next group's batched forward (three stages) spread between this
        # group's compositor launches, the previous group's backwards between
        bw = [("b", vg) for vg in pending_bwd]
        if k + 1 < len(groups):
            st_ = fwd_stepper(groups[k + 1])
            h = len(bw) // 2
            side = [("f", st_)] + bw[:h] + [("f", st_)] + bw[h:] + [("f", st_)]
        else:
            side = bw
        pending_bwd = []
        done = 0

        def run_side(upto):
            nonlocal done
            while done < upto:
                kind, x = side[done]
                if kind == "f":
                    x()
                else:
                    bwd(*x)
                done += 1

        prepared = {}

        def prep(i):
            li, (payload, _seg) = items[i]
            with torch.cuda.stream(fs):
                work = backend.prepare(gk[li], views[gk[li]], payload)
                ev = torch.cuda.Event()
                ev.record(fs)
            prepared[i] = (work, ev)

        grads = {}
        if items:
            prep(0)
        for i, (li, (payload, _seg)) in enumerate(items):
            v = gk[li]
            work, ev = prepared.pop(i)
            hold.append(work)
            main.wait_event(ev)
            t0 = _Stopwatch(payload.z.device)
            grads[li] = backend.render_prepared(v, views[v], work, images[v],
                                                None if priors is None else priors[v],
                                                None if normal_priors is None
                                                else normal_priors[v])
            timers[v] = t0.stop()
            _tr(f"r{v}")
            if i + 1 < len(items):
                prep(i + 1)
            _tr(f"p{v}")
            run_side((i + 1) * len(side) // len(items))
            _tr(f"s{v}")
        run_side(len(side))
        if k + 1 < len(groups):
            nxt = exchange(k + 1)
        main.wait_stream(ss)          # order main after this rank's NCCL issue on ss
        back = return_grads(plan, grads, backend.grad_like(), group)
        _tr(f"ret{k}")
        hold.append((grads, back))
        ts.wait_stream(main)          # the returned gradients
        pending_bwd = [(v, back[li]) for li, v in enumerate(gk)]
    for v, g in pending_bwd:
        bwd(v, g)
    _tr("bwd_last")
    for st in (ts, fs, ss):
        main.wait_stream(st)
    backend._hold = hold              # released by the next step's begin_step
    return timers


class _Stopwatch:
    """Seconds of the work issued between construction and stop(): CUDA
    events on the current stream for device work, wall clock otherwise."""

    def __init__(self, device):
        self.cuda = getattr(device, "type", "cpu") == "cuda"
        if self.cuda:
            self.a = torch.cuda.Event(enable_timing=True)
            self.b = torch.cuda.Event(enable_timing=True)
            self.a.record()
        else:
            import time
            self.t = time.perf_counter()

    def stop(self) -> "_Stopwatch":
        if self.cuda:
            self.b.record()
        else:
            import time
            self.t = time.perf_counter() - self.t
        return self

    def seconds(self) -> float:
        if self.cuda:
            self.b.synchronize()
            return self.a.elapsed_time(self.b) / 1e3
        return float(self.t)


def check_replicas(checksum: torch.Tensor, group=None) -> None:
    """Decoder replicas must stay bit-identical (reference trainer.py:204-207)."""
    lo, hi = checksum.clone(), checksum.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    if not torch.equal(lo, hi):
        raise ProtocolError("decoder replicas diverged across ranks")


# ------------------------------------------------------------------ CUDA backend

class CudaShardBackend:
    """Drives the sm_100a kernels for one rank of the sharded step."""

    def __init__(self, state, rank: int, world: int):
        from . import device as D
        self.D = D
        self.state = state
        self.rank, self.world = rank, world
        self._owned_key = None
        self.work: dict = {}
        self.timer = None     # optional trainer.GpuTimer for per-kernel spans
        self.isects = 0
        self.have, self.have_n = [], []

    @property
    def owned(self) -> torch.Tensor:
        """u8 mask of this rank's anchors (Eq. 3: i mod M per level), rebuilt
        whenever anchor growth changed the level sizes."""
        st = self.state
        key = tuple(lv.count for lv in st.scene.levels)
        if key != self._owned_key:
            owner = (st.assignment.flat_owner() if self.world == st.cfg.workers
                     else np.concatenate([np.arange(lv.count) % self.world
                                          for lv in st.scene.levels]))
            self._owned = (torch.as_tensor(owner) == self.rank).to(torch.uint8).cuda()
            self._owned_key = key
        return self._owned

    def schedule(self) -> tuple[float, float, float]:
        """(w2, w3, normal weight) of the current step (trainer.py:112-120)."""
        from .trainer import weight_schedule
        st = self.state
        w2, w3 = weight_schedule(st.step, st.cfg)
        return w2, w3, float(getattr(st.cfg, "normal_weight", 0.0))

    def begin_step(self, views, have=(), have_n=()) -> None:
        st = self.state
        self._hold = None             # the previous step's buffers (synced since)
        st.flat.grad.zero_()
        B = len(views)
        self.B = B
        self.have, self.have_n = list(have), list(have_n)
        self._hw = np.array([v.height * v.width * 3 for v in views], dtype=np.float64)
        self.sums = torch.zeros((B, 3), dtype=torch.float64, device="cuda")
        self.counts = torch.zeros((B, 2), dtype=torch.int32, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.work.clear()
        self.gaussians = 0
        self.geo = None
        # decoder weight image of this step's weights, shared by every view
        self._dimg = (self.D.decoder_image(st.params.abi(), st.n)
                      if self.D.use_tensor_cores(st.n) else None)
        self.isects = 0

    @property
    def deterministic(self) -> bool:
        return bool(getattr(self.state.cfg, "deterministic", False))

    def grad_like(self) -> torch.Tensor:
        return torch.zeros((0, self.D.GRAD_F32), dtype=torch.float32, device="cuda")

    def forward_shard(self, v: int, view) -> SplatPayload:
        D, st = self.D, self.state
        ds = st.dscene
        mask = ds.cull(view)
        active = D.select(mask & self.owned)
        an = st.anchors
        dec = D.decode(st.params.abi(), st.n, active, ds.centers, an.emb, an.log_scales,
                       an.offsets, view, ds.lod_ref, ds.max_scale, self.status, keep_cache=True,
                       img=self._dimg)
        self.gaussians += dec.count
        P = D.project(dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, view,
                      self.status)
        src = P.src.long()
        gid = active.long()[src // st.n] * st.n + src % st.n
        self.work[v] = (active, dec, P)
        return SplatPayload(P.rec, P.zkey.view(torch.float64), P.radius, gid)

    def prepare(self, v: int, view, payload: SplatPayload):
        """Merge the view's received splats in (z, gid) order and bin them."""
        D = self.D
        n = payload.count
        order = D.sort_z_gid(payload.z, payload.gid, int32=True)
        if isinstance(payload, PackedPayload):
            from ._lib import call, ptr, stream
            rs = torch.empty((max(n, 1), D.REC_F32), dtype=torch.float32, device="cuda")
            rr = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
            call("vsx_gather_splat_rows", c_void_p(payload.rows_ptr()), ptr(payload.rowmap),
                 ptr(order), n, ptr(rs), ptr(rr), stream())
            zk = payload.z.view(torch.int64)
            P = D.Projected(rs[:n], rr[:n], lambda: zk[order.long()], order, n)
            Bn = D.bin_tiles(P, view.width, view.height)
            return P, Bn, order
        # records and radii gathered in merge order by vsx_gather_splats (the
        # eager row gather took ~15x longer)
        P = D.gather_projected(payload.rec.contiguous(), payload.z.view(torch.int64),
                               payload.radius.contiguous(), order, n)
        Bn = D.bin_tiles(P, view.width, view.height)
        return P, Bn, order

    def forward_shards(self, vs: list[int], views):
        """forward_shard for a group of views with two host reads in total
        (all selection counts, then all kept counts) instead of two per view.
        A generator: each next() runs one stage, so a caller can interleave
        the stages with other host work; returns {v: SplatPayload}."""
        D, st = self.D, self.state
        ds = st.dscene
        an = st.anchors
        sel = []
        for v in vs:
            sel.append(D.select_async(ds.cull(views[v]) & self.owned))
        yield
        counts = torch.cat([c for _, c in sel]).cpu().tolist() if sel else []
        launched = []
        for v, (idx, _), c in zip(vs, sel, counts):
            active = idx[:c]
            dec = D.decode(st.params.abi(), st.n, active, ds.centers, an.emb, an.log_scales,
                           an.offsets, views[v], ds.lod_ref, ds.max_scale, self.status,
                           keep_cache=True, img=self._dimg)
            self.gaussians += dec.count
            launched.append((active, dec, D.project_launch(
                dec.means, dec.opacity, dec.color, dec.scale, dec.quat, dec.normal, views[v],
                self.status, sort=False)))
        yield
        kept = torch.cat([pl.kept for _, _, pl in launched]).cpu().tolist() if launched else []
        out = {}
        from ._lib import call, ptr, stream
        for v, (active, dec, pl), k in zip(vs, launched, kept):
            P = D.project_finish(pl, k if pl.g else 0)
            n = P.count
            gid = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")[:n]
            z = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")[:n]
            if n:
                call("vsx_payload_keys", ptr(active), ptr(P.src), ptr(pl.key), n, st.n,
                     ptr(gid), ptr(z), stream())
            self.work[v] = (active, dec, P)
            out[v] = SplatPayload(P.rec, z.view(torch.float64), P.radius, gid)
        return out

    def render(self, v: int, view, payload: SplatPayload, image, prior, nprior) -> torch.Tensor:
        return self.render_prepared(v, view, self.prepare(v, view, payload), image, prior, nprior)

    def _loss(self, v: int, view, image, prior, nprior, sums, counts, band=(0, 0)):
        """The fused objective of view v (or of its tile-row band) -> (desc, buffers)."""
        from ._lib import VsxLossDesc, ptr
        from .trainer import _mask_u8, _prior_arrays, _to_device_image, weight_schedule
        st = self.state
        H, W = view.height, view.width
        w2, _ = weight_schedule(st.step, st.cfg)
        wn = float(getattr(st.cfg, "normal_weight", 0.0))
        gt = _to_device_image(image, (H, W, 3))
        pd = pv = pn = pnv = None
        if v in self.have:
            d_, m_ = _prior_arrays(prior)
            pd, pv = _to_device_image(d_, (H, W)), _mask_u8(m_, (H, W))
        if v in self.have_n:
            pn, pnv = _to_device_image(nprior[0], (H, W, 3)), _mask_u8(nprior[1], (H, W))
        # the depth / normal terms are means over the views that carry a prior
        # (trainer.py:296-306, losses.py:84): normalised by that global count
        loss = VsxLossDesc(gt_rgb=gt.data_ptr(), prior_depth=ptr(pd),
                           prior_depth_valid=ptr(pv), prior_normal=ptr(pn),
                           prior_normal_valid=ptr(pnv), rgb_scale=1.0 / (self.B * H * W * 3),
                           depth_weight=w2 / len(self.have) if pd is not None else 0.0,
                           normal_weight=wn / len(self.have_n) / 3.0 if pn is not None else 0.0,
                           sums=sums.data_ptr(), counts=counts.data_ptr(),
                           tile_row0=int(band[0]), tile_rows=int(band[1]))
        return loss, (gt, pd, pv, pn, pnv)

    def render_prepared(self, v: int, view, work, image, prior, nprior) -> torch.Tensor:
        D, st = self.D, self.state
        P, Bn, order = work
        loss, keep = self._loss(v, view, image, prior, nprior, self.sums[v], self.counts[v])
        from .trainer import _span
        self.isects += Bn.intersections
        det = bool(getattr(st.cfg, "deterministic", False))
        with _span(self.timer, "raster_fwd"):
            R = D.raster_forward(P, Bn, view, loss=loss, deterministic=det)
        with _span(self.timer, "raster_bwd"):
            gs = D.raster_backward(P, Bn, view, R, loss=loss, deterministic=det)
        return _unsort_rows(gs, order)

    # ---- tile-row bands (a view split over renderer ranks when B < M)

    @staticmethod
    def band_rows(view, S: int) -> list[tuple[int, int]]:
        """S contiguous tile-row bands (row0, rows) of the view, sizes within one."""
        tyn = (view.height + 15) // 16
        S = max(1, min(S, tyn))
        cuts = [tyn * b // S for b in range(S + 1)]
        return [(cuts[b], cuts[b + 1] - cuts[b]) for b in range(S)]

    def band_payload(self, payload: SplatPayload, view, band):
        """The payload rows whose tile rectangle (renderer.py:216-221, float64
        floor as vsx_bin_*) reaches the band's tile rows, and their indices."""
        tyn = (view.height + 15) // 16
        if payload.count == 0:
            idx = torch.zeros(0, dtype=torch.int64, device=payload.z.device)
        else:
            yv = payload.rec.view(torch.float64)[:, 1]
            r = payload.radius
            y0 = torch.clamp(torch.floor((yv - r) * 0.0625), min=0.0)
            y1 = torch.clamp(torch.floor((yv + r) * 0.0625), max=float(tyn - 1))
            lo, hi = float(band[0]), float(band[0] + band[1] - 1)
            idx = torch.nonzero((y1 >= y0) & (y0 <= hi) & (y1 >= lo)).flatten()
        sub = SplatPayload(payload.rec[idx], payload.z[idx], payload.radius[idx],
                           payload.gid[idx])
        return sub, idx

    def begin_bands(self, n_items: int) -> None:
        self.isums = torch.zeros((n_items, 3), dtype=torch.float64, device="cuda")
        self.icounts = torch.zeros((n_items, 2), dtype=torch.int32, device="cuda")
        self.pending = {}

    def band_forward(self, it: int, v: int, view, work, image, prior, nprior, band) -> None:
        D, st = self.D, self.state
        P, Bn, order = work
        loss, keep = self._loss(v, view, image, prior, nprior, self.isums[it], self.icounts[it],
                                band)
        self.isects += Bn.intersections
        det = bool(getattr(st.cfg, "deterministic", False))
        R = D.raster_forward(P, Bn, view, loss=loss, deterministic=det)
        self.pending[it] = (work, view, loss, keep, R)

    def band_backward(self, it: int, extra=None) -> torch.Tensor:
        """The band's backward; ``extra`` = the view's NCC cotangents (rgb,
        normal, depth images) or None."""
        from ._lib import ptr
        D, st = self.D, self.state
        (P, Bn, order), view, loss, keep, R = self.pending.pop(it)
        if extra is not None:
            ex_rgb, ex_nrm, ex_dep = extra
            loss.extra_rgb, loss.extra_normal = ptr(ex_rgb), ptr(ex_nrm)
            loss.extra_depth = ptr(ex_dep)
            keep = (keep, extra)
        det = bool(getattr(st.cfg, "deterministic", False))
        gs = D.raster_backward(P, Bn, view, R, loss=loss, deterministic=det)
        return _unsort_rows(gs, order)

    def backward_shard(self, v: int, view, grads: torch.Tensor) -> None:
        from ._lib import call, ptr, stream
        from .decoder import decoder_backward_into
        D, st = self.D, self.state
        ds = st.dscene
        active, dec, P = self.work[v]
        gg = D.project_backward(dec.means, dec.scale, dec.quat, dec.normal, P,
                                grads.contiguous(), view)
        # growth pressure (trainer.py:341-349): every gaussian of an owned
        # anchor is decoded here, so the owner's sums are complete for its
        # anchors (sync_growth sums them across ranks before grow_anchors)
        call("vsx_growth_accumulate", ptr(gg["means"]), ptr(active), int(active.numel()), st.n,
             ptr(st.grow_sum_flat), ptr(st.grow_cnt_flat), stream())
        an, ag = st.anchors, st.anchor_grads
        decoder_backward_into(st.params, st.dgrads, active, ds.centers, an.emb, an.log_scales,
                              an.offsets, view, ds.lod_ref, ds.max_scale, dec, gg["means"],
                              gg["opacities"], gg["colors"], gg["scales"], gg["quats"],
                              gg["normals"], ag.emb, ag.log_scales, ag.offsets)

    def decoder_grad(self) -> torch.Tensor:
        st = self.state
        lo, hi = st.flat.group_spans["dec"]
        return st.flat.grad[lo:hi]

    def loss_terms(self) -> torch.Tensor:
        return torch.cat([self.sums, self.counts.double()], dim=1)

    def finish_step(self, losses: torch.Tensor) -> dict:
        from .errors import NumericalError
        from .trainer import weight_schedule
        st = self.state
        self.D.check_status(self.status, "sharded train_step")
        w2, _ = weight_schedule(st.step, st.cfg)
        L = losses.cpu().numpy()
        hw = self._hw
        rgb = float(np.mean(L[:, 0] / hw))
        dcnt, ncnt = L[:, 3], L[:, 4]
        dterm = np.where(dcnt > 0, L[:, 1] / np.maximum(dcnt, 1), 0.0)
        nterm = np.where(ncnt > 0, L[:, 2] / (3 * np.maximum(ncnt, 1)), 0.0)
        depth = float(np.mean(dterm[self.have])) if self.have else 0.0
        normal = float(np.mean(nterm[self.have_n])) if self.have_n else 0.0
        w3 = weight_schedule(st.step, st.cfg)[1]
        geo = self.geo[0] if self.geo is not None else 0.0
        total = rgb + w2 * depth + float(getattr(st.cfg, "normal_weight", 0.0)) * normal + \
            w3 * geo
        if not np.isfinite(total):
            raise NumericalError(f"non-finite loss at step {st.step}")
        st.adam()
        st.step += 1
        out = {"total": total, "rgb": rgb, "depth": depth, "normal": normal, "geo": geo,
               "gaussians": self.gaussians}
        if self.geo is not None:
            out["geo_pairs"], out["geo_patches"] = self.geo[1].pairs_used, self.geo[1].patches_used
        return out

    def decoder_checksum(self) -> torch.Tensor:
        g = self.state.flat
        lo, hi = g.group_spans["dec"]
        return g.param[lo:hi].view(torch.int32).long().sum().reshape(1)


def sync_growth(state, group=None) -> None:
    """Sum the per-anchor growth accumulators over the ranks (each owner holds
    the complete sums of its own anchors), so every rank's grow_anchors makes
    the same decisions with the same RNG draws (trainer.py:379-454)."""
    dist.all_reduce(state.grow_sum_flat, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(state.grow_cnt_flat, op=dist.ReduceOp.SUM, group=group)
