"""Float64 CPU restatement of the voxsplat training step (test oracle only).

Every function cites the reference lines it restates (paths relative to
``/root/reference/pkg/src/voxsplat``). Differentiable pieces are torch
float64 so gradients come from autograd, exactly as in the reference
(``trainer.py:323-339``); integer/bookkeeping pieces (culling decisions,
z-sort, tile binning) are numpy.

Structure differs from the reference only where it bounds memory without
changing the math: rasterisation runs tile by tile, and a view's backward
runs right after its forward (the batch loss is a sum of per-view terms, so
accumulating per-view gradients equals the reference's single autograd
call up to float64 summation order).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

F64 = torch.float64

# renderer.py:39-47, decoder.py:27-30, scene.py:23-24, partition.py:22
Z_NEAR = 0.01
ALPHA_CLAMP = 0.99
EARLY_STOP_T = 1e-4
ALPHA_VALID_MIN = 1e-4
DENOM_GUARD = 1e-6
LOWPASS = 0.3
PATCH = 16
MIN_SCALE = 1e-6
HIDDEN = 64
EMBED_DIM = 32
IN_DIM = EMBED_DIM + 4
FRUSTUM_MARGIN = 0.10
HEADS = ("opacity", "color", "cov")
HEAD_WIDTH = {"opacity": 1, "color": 3, "cov": 7}
ADAM_EPS = 1e-15


@dataclass(frozen=True)
class Cam:
    """Plain camera record; build from any object with CameraView fields."""

    r: np.ndarray
    t: np.ndarray
    center: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    @classmethod
    def of(cls, view) -> "Cam":
        return cls(np.asarray(view.r, np.float64), np.asarray(view.t, np.float64),
                   np.asarray(view.center, np.float64), float(view.fx), float(view.fy),
                   float(view.cx), float(view.cy), int(view.width), int(view.height))

    @property
    def tiles(self) -> tuple[int, int]:
        return (self.width + PATCH - 1) // PATCH, (self.height + PATCH - 1) // PATCH


# ---------------------------------------------------------------- K1: culling

def cull(centers: np.ndarray, levels: np.ndarray, lod_count: int, lod_ref: float,
         lod_bias: int, cam: Cam) -> np.ndarray:
    """Active-anchor mask over level-major flat anchors.

    Restates ``scene.py:239-259`` (padded frustum test on the voxel centre)
    and ``scene.py:232-236`` (LoD = clip(floor(log2(ref/d) + bias), 0, K-1)),
    evaluated on the concatenation of all levels at once.
    """
    centers = np.asarray(centers, np.float64).reshape(-1, 3)
    if centers.shape[0] == 0:
        return np.zeros(0, dtype=bool)
    pc = centers @ cam.r.T + cam.t
    z = pc[:, 2]
    front = z > 1e-9
    zsafe = np.where(front, z, 1.0)
    u = np.where(front, cam.fx * pc[:, 0] / zsafe + cam.cx, -1e9)
    v = np.where(front, cam.fy * pc[:, 1] / zsafe + cam.cy, -1e9)
    mx, my = FRUSTUM_MARGIN * cam.width, FRUSTUM_MARGIN * cam.height
    inside = front & (u >= -mx) & (u <= cam.width + mx) & (v >= -my) & (v <= cam.height + my)
    dist = np.maximum(np.linalg.norm(centers - cam.center, axis=1), 1e-12)
    lod = np.clip(np.floor(np.log2(lod_ref / dist) + lod_bias), 0, lod_count - 1)
    return inside & (lod.astype(np.int64) == np.asarray(levels))


# ---------------------------------------------------------------- K2: decode

def decoder_init(n: int, seed: int = 0, scale_bias: float | None = None) -> dict:
    """Seeded decoder weights, same draw order as ``decoder.py:54-78``."""
    rng = np.random.default_rng(seed)
    out = {}
    for h in HEADS:
        width = HEAD_WIDTH[h] * n
        a1, a2 = 1.0 / np.sqrt(IN_DIM), 1.0 / np.sqrt(HIDDEN)
        out[f"{h}_w1"] = rng.uniform(-a1, a1, (IN_DIM, HIDDEN))
        out[f"{h}_b1"] = np.zeros(HIDDEN)
        out[f"{h}_w2"] = rng.uniform(-a2, a2, (HIDDEN, width))
        out[f"{h}_b2"] = np.zeros(width)
    if scale_bias is not None:
        out["cov_b2"].reshape(n, 7)[:, 0:3] = float(scale_bias)
    return out


def quat_rot(q: torch.Tensor) -> torch.Tensor:
    """(…,4) unit quaternion -> (…,3,3), ``decoder.py:108-114``."""
    w, x, y, z = q.unbind(-1)
    m = [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]
    return torch.stack(m, -1).reshape(*q.shape[:-1], 3, 3)


def decode(weights: dict, centers, emb, scales, offsets, cam_center, lod_ref: float,
           max_scale: float, n: int) -> dict:
    """Anchor -> n gaussians (``decoder.py:142-180``), all (V, n, …) float64.

    Input block x = [emb | d/ref | (c - cam)/d] with d = max(|c - cam|, 1e-12);
    three tanh MLP heads 36 -> 64 -> {n, 3n, 7n}; sigmoid opacity/colour;
    scale = clamp(exp(raw), 1e-6, max_scale); q = normalise(raw + (1,0,0,0));
    mean = c + offset * l_v; normal = column argmin(scale) of R(q).
    """
    c = torch.as_tensor(centers, dtype=F64)
    v = c.shape[0]
    rel = c - torch.as_tensor(np.asarray(cam_center, np.float64))
    d = torch.linalg.norm(rel, dim=-1, keepdim=True).clamp_min(1e-12)
    x = torch.cat([emb, d / lod_ref, rel / d], dim=-1)
    raw = {}
    for h in HEADS:
        hid = torch.tanh(x @ weights[f"{h}_w1"] + weights[f"{h}_b1"])
        raw[h] = hid @ weights[f"{h}_w2"] + weights[f"{h}_b2"]
    opac = torch.sigmoid(raw["opacity"]).reshape(v, n)
    col = torch.sigmoid(raw["color"]).reshape(v, n, 3)
    cov = raw["cov"].reshape(v, n, 7)
    s = torch.clamp(torch.exp(cov[..., 0:3]), MIN_SCALE, max_scale)
    qr = cov[..., 3:7] + torch.tensor([1.0, 0.0, 0.0, 0.0], dtype=F64)
    q = qr / torch.linalg.norm(qr, dim=-1, keepdim=True).clamp_min(1e-12)
    means = c.unsqueeze(1) + offsets * scales.unsqueeze(1)
    rot = quat_rot(q)
    axis = torch.argmin(s, dim=-1)
    normal = torch.take_along_dim(rot, axis[..., None, None].expand(v, n, 3, 1), dim=-1)
    return {"means": means, "opacities": opac, "colors": col, "scales": s,
            "quats": q, "normals": normal.squeeze(-1)}


def leaf_gaussians(means, opacities, colors, scales, quats, requires_grad=False) -> dict:
    """Raw gaussian leaves -> projectable dict (``renderer.py:110-141``).

    Quaternions are normalised (norm clamped at 1e-12) and the normal is the
    rotation column of the smallest scale. Leaves are returned under "leaves".
    """
    leaves = {k: torch.tensor(np.asarray(a, np.float64)) for k, a in
              (("means", means), ("opacities", opacities), ("colors", colors),
               ("scales", scales), ("quats", quats))}
    leaves["means"] = leaves["means"].reshape(-1, 3)
    leaves["colors"] = leaves["colors"].reshape(-1, 3)
    leaves["scales"] = leaves["scales"].reshape(-1, 3)
    leaves["quats"] = leaves["quats"].reshape(-1, 4)
    leaves["opacities"] = leaves["opacities"].reshape(-1)
    if requires_grad:
        for t in leaves.values():
            t.requires_grad_(True)
    q = leaves["quats"] / torch.linalg.norm(leaves["quats"], dim=-1, keepdim=True).clamp_min(1e-12)
    rot = quat_rot(q)
    axis = torch.argmin(leaves["scales"], dim=-1)
    nrm = torch.take_along_dim(rot, axis[:, None, None].expand(-1, 3, 1), -1).squeeze(-1)
    return {"means": leaves["means"], "opacities": leaves["opacities"],
            "colors": leaves["colors"], "scales": leaves["scales"], "quats": q,
            "normals": nrm, "leaves": leaves}


def flatten_decoded(dec: dict) -> dict:
    return {k: t.reshape(-1, *t.shape[2:]) for k, t in dec.items()}


# ---------------------------------------------------------------- K3: project

def project(g: dict, gid: np.ndarray, cam: Cam) -> dict:
    """EWA projection + (z, gid) sort, ``renderer.py:144-204``.

    Returns the sorted screen-space splats (torch, graph-connected) and the
    numpy bookkeeping: ``src`` (index into g for each sorted splat), ``zkey``,
    ``radius``, ``gid``.
    """
    R = torch.as_tensor(cam.r, dtype=F64)
    t = torch.as_tensor(cam.t, dtype=F64)
    mu_all = g["means"] @ R.T + t
    keep = np.flatnonzero(mu_all[:, 2].detach().numpy() > Z_NEAR)
    kt = torch.from_numpy(keep)
    mu = mu_all[kt]
    gid = np.asarray(gid)[keep]
    x, y, z = mu.unbind(-1)
    mean2d = torch.stack([cam.fx * x / z + cam.cx, cam.fy * y / z + cam.cy], -1)
    rq = quat_rot(g["quats"][kt])
    s2 = g["scales"][kt] ** 2
    cov_w = rq @ (s2.unsqueeze(-1) * rq.transpose(-1, -2))
    cov_c = R @ cov_w @ R.T
    jac = torch.zeros((len(keep), 2, 3), dtype=F64)
    zi = 1.0 / z
    jac[:, 0, 0] = cam.fx * zi
    jac[:, 0, 2] = -cam.fx * x * zi * zi
    jac[:, 1, 1] = cam.fy * zi
    jac[:, 1, 2] = -cam.fy * y * zi * zi
    cov2 = jac @ cov_c @ jac.transpose(-1, -2)
    a = cov2[:, 0, 0] + LOWPASS
    b = cov2[:, 0, 1]
    c = cov2[:, 1, 1] + LOWPASS
    det = a * c - b * b
    if len(keep) and bool((det.detach() <= 0).any()):
        raise FloatingPointError("non positive definite 2d covariance")
    conic = torch.stack([c / det, -b / det, a / det], -1)
    lam = 0.5 * (a + c) + torch.sqrt(torch.clamp(0.25 * (a - c) ** 2 + b * b, min=0.0))
    radius = (3.0 * torch.sqrt(lam)).detach().numpy()
    n_cam = g["normals"][kt] @ R.T
    facing = torch.sign((n_cam * mu).sum(-1)).detach()
    n_cam = n_cam * torch.where(facing > 0, -1.0, 1.0).to(F64).unsqueeze(-1)
    plane_d = (n_cam * mu).sum(-1)
    zkey = z.detach().numpy()
    order = np.lexsort((gid, zkey))
    o = torch.from_numpy(order)
    return {"mean2d": mean2d[o], "conic": conic[o], "color": g["colors"][kt][o],
            "opacity": g["opacities"][kt][o], "normal_cam": n_cam[o],
            "plane_d": plane_d[o], "radius": radius[order], "zkey": zkey[order],
            "gid": gid[order], "src": keep[order]}


# ---------------------------------------------------------------- K4: binning

def bin_tiles(mean2d: np.ndarray, radius: np.ndarray, width: int, height: int):
    """Per-tile ascending splat lists, ``renderer.py:207-226``.

    Returns (offsets[T+1], lists[I]) CSR. A splat covers tiles
    x in [max(floor((u-r)/16), 0), min(floor((u+r)/16), tx-1)] (same for y);
    empty rectangles are skipped. Lists hold sorted-splat indices ascending.
    """
    tx_n, ty_n = (width + PATCH - 1) // PATCH, (height + PATCH - 1) // PATCH
    mean2d = np.asarray(mean2d, np.float64).reshape(-1, 2)
    r = np.asarray(radius, np.float64)
    u, v = mean2d[:, 0], mean2d[:, 1]
    x0 = np.maximum(np.floor((u - r) / PATCH), 0.0)
    x1 = np.minimum(np.floor((u + r) / PATCH), tx_n - 1.0)
    y0 = np.maximum(np.floor((v - r) / PATCH), 0.0)
    y1 = np.minimum(np.floor((v + r) / PATCH), ty_n - 1.0)
    ok = (x1 >= x0) & (y1 >= y0)
    idx = np.flatnonzero(ok)
    x0i, x1i = x0[idx].astype(np.int64), x1[idx].astype(np.int64)
    y0i, y1i = y0[idx].astype(np.int64), y1[idx].astype(np.int64)
    w = x1i - x0i + 1
    cnt = w * (y1i - y0i + 1)
    total = int(cnt.sum())
    owner = np.repeat(np.arange(idx.size), cnt)
    local = np.arange(total) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    tile = (y0i[owner] + local // w[owner]) * tx_n + (x0i[owner] + local % w[owner])
    perm = np.argsort(tile, kind="stable")
    lists = idx[owner[perm]].astype(np.int64)
    offsets = np.concatenate([[0], np.cumsum(np.bincount(tile, minlength=tx_n * ty_n))])
    return offsets.astype(np.int64), lists


# ---------------------------------------------------------------- K5: raster

def _tile_pixels(tx: int, ty: int):
    dv, du = np.divmod(np.arange(PATCH * PATCH), PATCH)
    return (tx * PATCH + du).astype(np.float64), (ty * PATCH + dv).astype(np.float64)


def raster_tile(S: dict, idx: np.ndarray, tx: int, ty: int, cam: Cam,
                jitter: torch.Generator | None = None) -> dict:
    """One 16x16 tile, all 256 pixels (ragged ones included).

    Blend = ``renderer.py:242-279``: power at integer pixel coordinates,
    alpha = min(o * exp(min(power, 0)), 0.99), T = prefix product of
    (1 - alpha), live = T_prev >= 1e-4 (detached), w = alpha * T_prev * live,
    accumulated alpha / rgb / raw normal / plane offset, and
    denom = raw_normal . ((u - cx)/fx, (v - cy)/fy, 1).
    Finalize = ``renderer.py:282-301``.

    ``jitter`` (tests only) multiplies the per-(splat, pixel) power, each
    transmittance factor and each weight by independent (1 + 2^-23 u),
    u ~ U(-1, 1): float32 rounding of every intermediate, so that
    |g - g_jitter| estimates a gradient element's float32 floor.
    """
    pu_np, pv_np = _tile_pixels(tx, ty)
    pu, pv = torch.from_numpy(pu_np), torch.from_numpy(pv_np)
    it = torch.from_numpy(np.asarray(idx, np.int64))
    m = S["mean2d"][it]
    con = S["conic"][it]
    dx = pu.unsqueeze(0) - m[:, 0:1]
    dy = pv.unsqueeze(0) - m[:, 1:2]

    def jit(x):
        if jitter is None:
            return x
        u = torch.rand(x.shape, generator=jitter, dtype=F64) * 2.0 - 1.0
        return x * (1.0 + 2.0 ** -23 * u)
    power = jit(-0.5 * (con[:, 0:1] * dx * dx + 2.0 * con[:, 1:2] * dx * dy
                        + con[:, 2:3] * dy * dy))
    alpha = S["opacity"][it].unsqueeze(-1) * torch.exp(torch.clamp(power, max=0.0))
    alpha = torch.clamp(alpha, max=ALPHA_CLAMP)
    trans = torch.cumprod(jit(1.0 - alpha), dim=0)
    t_prev = torch.cat([torch.ones_like(trans[:1]), trans[:-1]], dim=0)
    live = (t_prev >= EARLY_STOP_T).to(F64).detach()
    w = jit(alpha * t_prev * live)                              # (L, 256)
    acc = w.sum(0)
    rgb = w.transpose(0, 1) @ S["color"][it]
    raw_n = jit(w.transpose(0, 1) @ S["normal_cam"][it])
    dist = jit((w * S["plane_d"][it].unsqueeze(-1)).sum(0))
    rx = (pu - cam.cx) / cam.fx
    ry = (pv - cam.cy) / cam.fy
    denom = jit(raw_n[:, 0] * rx + raw_n[:, 1] * ry + raw_n[:, 2])
    covered = acc >= ALPHA_VALID_MIN
    valid = covered & (denom.abs() >= DENOM_GUARD)
    depth = torch.where(valid, dist / torch.where(valid, denom, torch.ones_like(denom)),
                        torch.zeros_like(denom))
    nrm = torch.linalg.norm(raw_n, dim=-1, keepdim=True).clamp_min(1e-12)
    normal = torch.where(covered.unsqueeze(-1), raw_n / nrm, torch.zeros_like(raw_n))
    nlive = live.sum(0).long()
    last = trans.gather(0, (nlive - 1).clamp_min(0).unsqueeze(0)).squeeze(0)
    t_final = torch.where(nlive > 0, last, torch.ones_like(acc)).detach()
    return {"rgb": rgb, "alpha": acc, "raw_normal": raw_n, "dist": dist, "denom": denom,
            "depth": depth, "normal": normal, "valid": valid.detach(),
            "t_final": t_final, "n_contrib": nlive.to(F64)}


IMAGE_KEYS = ("rgb", "alpha", "raw_normal", "dist", "denom", "depth", "normal",
              "valid", "t_final", "n_contrib")


def raster(S: dict, offsets: np.ndarray, lists: np.ndarray, cam: Cam) -> dict:
    """Whole view (``renderer.py:390-449``), graph-connected to S.

    Tiles with empty lists stay zero / invalid; ragged pixels are dropped.
    """
    tx_n, ty_n = cam.tiles
    H, W = cam.height, cam.width
    parts = {k: [] for k in IMAGE_KEYS}
    sel = []
    for t in range(tx_n * ty_n):
        lo, hi = int(offsets[t]), int(offsets[t + 1])
        if hi == lo:
            continue
        ty, tx = divmod(t, tx_n)
        out = raster_tile(S, lists[lo:hi], tx, ty, cam)
        pu, pv = _tile_pixels(tx, ty)
        inside = (pu < W) & (pv < H)
        keep = torch.from_numpy(np.flatnonzero(inside))
        for k in IMAGE_KEYS:
            parts[k].append(out[k][keep])
        sel.append((pv[inside] * W + pu[inside]).astype(np.int64))
    shapes = {"rgb": 3, "raw_normal": 3, "normal": 3}
    res = {}
    index = torch.from_numpy(np.concatenate(sel)) if sel else None
    for k in IMAGE_KEYS:
        c = shapes.get(k)
        dtype = torch.bool if k == "valid" else F64
        base = torch.zeros((H * W, c) if c else (H * W,), dtype=dtype)
        if k == "t_final":
            base = torch.ones(H * W, dtype=F64)
        if index is not None:
            base = base.index_copy(0, index, torch.cat(parts[k]))
        res[k] = base.reshape((H, W, c) if c else (H, W))
    res["counts"] = np.diff(offsets)
    return res


# ---------------------------------------------------------------- K9: losses

def l1_loss(rendered: list, reference: list) -> torch.Tensor:
    """``losses.py:43-53``: mean over views of mean |I_hat - I|."""
    terms = [(r - torch.as_tensor(np.asarray(g, np.float64))).abs().mean()
             for r, g in zip(rendered, reference)]
    return torch.stack(terms).mean()


def depth_l1_loss(depths, rvalid, priors, pvalid):
    """``losses.py:65-84``: masked L1 per view over supervised pixels, mean over views."""
    terms, total = [], 0
    for d, rv, p, pv in zip(depths, rvalid, priors, pvalid):
        mask = (torch.as_tensor(np.asarray(pv, bool)) & torch.as_tensor(rv)).to(F64)
        cnt = int(mask.sum())
        total += cnt
        if cnt == 0:
            terms.append(torch.zeros((), dtype=F64))
        else:
            terms.append(((d - torch.as_tensor(np.asarray(p, np.float64))).abs() * mask).sum() / cnt)
    return torch.stack(terms).mean(), total


# ---------------------------------------------------------------- K10: Adam

def cosine_lr(step: int, base: float, total_steps: int, final_factor: float) -> float:
    """``trainer.py:123-125``."""
    lo = base * final_factor
    return lo + 0.5 * (base - lo) * (1.0 + np.cos(np.pi * step / total_steps))


def adam_update(p: torch.Tensor, g: torch.Tensor, m: torch.Tensor, v: torch.Tensor,
                step: int, lr: float, b1: float = 0.9, b2: float = 0.999) -> None:
    """In-place Adam with bias correction, ``trainer.py:220-229`` (+ add to p)."""
    t = step + 1
    with torch.no_grad():
        m.mul_(b1).add_(g, alpha=1 - b1)
        v.mul_(b2).addcmul_(g, g, value=1 - b2)
        p.add_(-lr * (m / (1 - b1 ** t)) / ((v / (1 - b2 ** t)).sqrt() + ADAM_EPS))


def weight_schedule(step: int, total: int, s2: int, s3: int, w3_max: float = 0.2):
    """``trainer.py:112-120``."""
    w2 = 1.0 - (step - s2) / (total - s2) if step >= s2 and total > s2 else 0.0
    w3 = w3_max * (step - s3) / (total - s3) if step >= s3 and total > s3 else 0.0
    return w2, w3


# ---------------------------------------------------------------- train step

@dataclass
class OracleState:
    """Float64 training state over level-major flat anchors.

    Mirrors ``TrainState`` (``trainer.py:159-247``): decoder leaves, per-anchor
    embeddings / log-scales / offsets, Adam moments, step counter.
    """

    centers: np.ndarray
    levels: np.ndarray
    lod_count: int
    lod_ref: float
    lod_bias: int
    base_voxel_size: float
    n: int
    weights: dict
    emb: torch.Tensor
    log_scales: torch.Tensor
    offsets: torch.Tensor
    total_steps: int = 100
    step2_start: int = 100
    step3_start: int = 100
    lr_decoder: float = 2e-3
    lr_embeddings: float = 5e-3
    lr_offsets: float = 1e-2
    lr_scales: float = 5e-3
    lr_final_factor: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    step: int = 0
    moments: dict = field(default_factory=dict)
    last_grads: dict = field(default_factory=dict)
    last_timing: dict = field(default_factory=dict)

    @classmethod
    def create(cls, centers, levels, lod_count, lod_ref, lod_bias, base_voxel_size, n,
               weights, emb, log_scales, offsets, **cfg) -> "OracleState":
        w = {k: torch.tensor(np.asarray(a, np.float64)) for k, a in weights.items()}
        st = cls(np.asarray(centers, np.float64), np.asarray(levels), lod_count, lod_ref,
                 lod_bias, base_voxel_size, n, w,
                 torch.tensor(np.asarray(emb, np.float64)),
                 torch.tensor(np.asarray(log_scales, np.float64)),
                 torch.tensor(np.asarray(offsets, np.float64)), **cfg)
        for name, p in st.params().items():
            st.moments[name] = (torch.zeros_like(p), torch.zeros_like(p))
        return st

    def params(self) -> dict:
        out = {f"dec/{k}": t for k, t in self.weights.items()}
        out.update({"emb": self.emb, "log_scales": self.log_scales, "offsets": self.offsets})
        return out

    def lr_for(self, name: str) -> float:
        base = {"emb": self.lr_embeddings, "log_scales": self.lr_scales,
                "offsets": self.lr_offsets}.get(name, self.lr_decoder)   # dec/* -> decoder
        return cosine_lr(self.step, base, self.total_steps, self.lr_final_factor)


def _view_splats(st: OracleState, cam: Cam, grad: bool):
    """Cull + decode + project one view; returns (projected dict, active idx)."""
    active = np.flatnonzero(cull(st.centers, st.levels, st.lod_count, st.lod_ref,
                                 st.lod_bias, cam))
    at = torch.from_numpy(active)
    ctx = torch.enable_grad() if grad else torch.no_grad()
    with ctx:
        dec = decode(st.weights, st.centers[active], st.emb[at], torch.exp(st.log_scales[at]),
                     st.offsets[at], cam.center, st.lod_ref, 3.0 * st.base_voxel_size, st.n)
        flat = flatten_decoded(dec)
        gid = (active[:, None] * st.n + np.arange(st.n)).reshape(-1)
        P = project(flat, gid, cam)
    return P, active, flat


SPLAT_KEYS = ("mean2d", "conic", "color", "opacity", "normal_cam", "plane_d")


def render_view(st: OracleState, cam: Cam) -> dict:
    """Forward-only render (``renderer.py:480-493``)."""
    with torch.no_grad():
        P, active, flat = _view_splats(st, cam, grad=False)
        offsets, lists = bin_tiles(P["mean2d"].numpy(), P["radius"], cam.width, cam.height)
        img = raster(P, offsets, lists, cam)
    img["splats"], img["offsets"], img["lists"], img["active"] = P, offsets, lists, active
    img["decoded"] = flat
    return img


def normal_l1_loss(normals, rvalid, priors, pvalid):
    """Normal-prior L1 of the RGB-D-N objective (the B200 build's "N" term).

    The reference has no standalone normal loss: it supervises normals only
    through the depth quotient (``renderer.py:276-278``) and Eq. 10
    (``losses.py:196-287``); SURVEY.md §8(d) cfg2 asks for an "N" term. This
    is its contract, written in the shape of Eq. 9 (``losses.py:65-84``): per
    view the mean of |n_hat - n_prior| over the 3 channels of the pixels that
    are depth-valid and prior-valid, then the mean over the views that have a
    prior. Returns (loss, supervised pixel count).
    """
    terms, total = [], 0
    for n, rv, p, pv in zip(normals, rvalid, priors, pvalid):
        mask = (torch.as_tensor(np.asarray(pv, bool)) & torch.as_tensor(rv)).to(F64)
        cnt = int(mask.sum())
        total += cnt
        if cnt == 0:
            terms.append(torch.zeros((), dtype=F64))
        else:
            d = (n - torch.as_tensor(np.asarray(p, np.float64))).abs().sum(-1)
            terms.append((d * mask).sum() / (3.0 * cnt))
    return torch.stack(terms).mean(), total


def train_step(st: OracleState, cams: list, images: list, priors: list | None = None,
               tile_limit: int | None = None, normal_priors: list | None = None,
               normal_weight: float = 0.0) -> dict:
    """One step over a batch of views (``trainer.py:258-376``, RGB + depth terms).

    ``priors`` (optional) is a list of (depth, valid) per view for the Eq. 9
    term, weighted by the stage schedule. ``normal_priors`` (optional,
    (normals, valid) per view) add ``normal_weight`` x the normal-prior L1
    (:func:`normal_l1_loss`). ``tile_limit`` renders only an evenly spaced
    sample of N non-empty tiles per view (bounded CPU-baseline sample); it is
    None for parity runs.
    """
    B = len(cams)
    w2, _ = weight_schedule(st.step, st.total_steps, st.step2_start, st.step3_start)
    use_depth = priors is not None and w2 > 0 and any(p is not None for p in priors)
    use_normal = normal_priors is not None and normal_weight > 0
    for p in [*st.weights.values(), st.emb, st.log_scales, st.offsets]:
        p.requires_grad_(True)
        p.grad = None
    have = [i for i in range(B) if use_depth and priors[i] is not None]
    have_n = [i for i in range(B) if use_normal and normal_priors[i] is not None]
    normal_terms = []
    rgb_terms, depth_terms, supervised, gaussians, max_tile = [], [], 0, 0, 0
    timing = {"t_fixed": 0.0, "t_tiles": 0.0, "tiles_done": 0, "tiles_nonempty": 0}
    for vi, cam in enumerate(cams):
        tv = time.perf_counter()
        P, active, flat = _view_splats(st, cam, grad=True)
        gaussians += flat["means"].shape[0]
        offsets, lists = bin_tiles(P["mean2d"].detach().numpy(), P["radius"],
                                   cam.width, cam.height)
        counts = np.diff(offsets)
        max_tile = max(max_tile, int(counts.max()) if counts.size else 0)
        leaves = {k: P[k].detach().clone().requires_grad_(True) for k in SPLAT_KEYS}
        gt = torch.as_tensor(np.asarray(images[vi], np.float64))
        H, W = cam.height, cam.width
        dnorm, prior_d, prior_v = 0.0, None, None
        nnorm, prior_n, prior_nv = 0.0, None, None
        full = None
        if vi in have or vi in have_n:
            with torch.no_grad():
                full = raster(leaves, offsets, lists, cam)
        if vi in have:
            prior_d = torch.as_tensor(np.asarray(priors[vi][0], np.float64))
            prior_v = torch.as_tensor(np.asarray(priors[vi][1], bool))
            cnt = int((prior_v & full["valid"]).sum())
            supervised += cnt
            dnorm = (w2 / len(have) / cnt) if cnt else 0.0
        if vi in have_n:
            prior_n = torch.as_tensor(np.asarray(normal_priors[vi][0], np.float64))
            prior_nv = torch.as_tensor(np.asarray(normal_priors[vi][1], bool))
            ncnt = int((prior_nv & full["valid"]).sum())
            nnorm = (normal_weight / len(have_n) / (3.0 * ncnt)) if ncnt else 0.0
        tx_n, ty_n = cam.tiles
        rgb_sum = torch.zeros((), dtype=F64)
        dep_sum = torch.zeros((), dtype=F64)
        nrm_sum = torch.zeros((), dtype=F64)
        done = 0
        timing["tiles_nonempty"] += int((np.diff(offsets) > 0).sum())
        tt = time.perf_counter()
        timing["t_fixed"] += tt - tv
        busy = np.flatnonzero(np.diff(offsets) > 0)
        if tile_limit is not None and busy.size > tile_limit:
            # evenly spaced sample of the non-empty tiles (bounded CPU baseline)
            busy = busy[np.linspace(0, busy.size - 1, tile_limit).round().astype(np.int64)]
        timing["isect_sampled"] = timing.get("isect_sampled", 0) + int(
            np.diff(offsets)[busy].sum())
        timing["isect_total"] = timing.get("isect_total", 0) + int(offsets[-1])
        for t in busy:
            lo, hi = int(offsets[t]), int(offsets[t + 1])
            done += 1
            ty, tx = divmod(t, tx_n)
            out = raster_tile(leaves, lists[lo:hi], tx, ty, cam)
            pu, pv = _tile_pixels(tx, ty)
            inside = np.flatnonzero((pu < W) & (pv < H))
            py, px = pv[inside].astype(np.int64), pu[inside].astype(np.int64)
            ki = torch.from_numpy(inside)
            diff = (out["rgb"][ki] - gt[py, px]).abs().sum()
            obj = diff / (B * H * W * 3)
            rgb_sum = rgb_sum + diff.detach()
            if prior_d is not None and dnorm:
                msk = (prior_v[py, px] & out["valid"][ki]).to(F64)
                dd = ((out["depth"][ki] - prior_d[py, px]).abs() * msk).sum()
                obj = obj + dnorm * dd
                dep_sum = dep_sum + dd.detach()
            if prior_n is not None and nnorm:
                msk = (prior_nv[py, px] & out["valid"][ki]).to(F64)
                nd = ((out["normal"][ki] - prior_n[py, px]).abs().sum(-1) * msk).sum()
                obj = obj + nnorm * nd
                nrm_sum = nrm_sum + nd.detach()
            if obj.requires_grad:
                obj.backward()
        tb = time.perf_counter()
        timing["t_tiles"] += tb - tt
        timing["tiles_done"] += done
        if tile_limit is None:
            # tiles without splats render black (renderer.py:390-449): their
            # pixels still count |0 - I| in the L1 term (no gradient)
            empty = np.flatnonzero(np.diff(offsets) == 0)
            if empty.size:
                ey, ex = np.divmod(empty, tx_n)
                m = np.zeros((ty_n * 16, tx_n * 16), bool)
                for y0, x0 in zip(ey * 16, ex * 16):
                    m[y0:y0 + 16, x0:x0 + 16] = True
                rgb_sum = rgb_sum + gt[torch.from_numpy(m[:H, :W])].abs().sum()
        rgb_terms.append(rgb_sum / (H * W * 3))
        if vi in have:
            depth_terms.append(dep_sum * (dnorm * len(have) / w2))
        if vi in have_n:
            normal_terms.append(nrm_sum * (nnorm * len(have_n) / normal_weight))
        grads = [leaves[k].grad if leaves[k].grad is not None else torch.zeros_like(leaves[k])
                 for k in SPLAT_KEYS]
        torch.autograd.backward([P[k] for k in SPLAT_KEYS], grads)
        timing["t_fixed"] += time.perf_counter() - tb
    st.last_timing = timing
    rgb = torch.stack(rgb_terms).mean()
    depth = torch.stack(depth_terms).mean() if depth_terms else torch.zeros((), dtype=F64)
    normal = torch.stack(normal_terms).mean() if normal_terms else torch.zeros((), dtype=F64)
    total = rgb + w2 * depth + normal_weight * normal
    if not bool(torch.isfinite(total)):
        raise FloatingPointError(f"non-finite loss at step {st.step}")
    st.last_grads = {}
    for name, p in st.params().items():
        g = p.grad if p.grad is not None else torch.zeros_like(p)
        st.last_grads[name] = g.clone()
        m, v = st.moments[name]
        adam_update(p.data, g, m, v, st.step, st.lr_for(name), st.beta1, st.beta2)
    report = {"step": st.step, "total": float(total), "rgb": float(rgb),
              "depth": float(depth), "normal": float(normal), "w2": w2, "gaussians": gaussians,
              "supervised_depth_px": supervised, "max_tile_splats": max_tile}
    st.step += 1
    for p in [*st.weights.values(), st.emb, st.log_scales, st.offsets]:
        p.requires_grad_(False)
        p.grad = None
    return report
