"""Float64 oracle backend for the sharded step (TEST INFRASTRUCTURE ONLY).

Implements the backend interface of ``paper_2503_23044_b200.dist`` with the
oracle's own functions (``oracle/pipeline.py``), so ``tests/test_dist_gloo.py``
can run the real C1/C2 routing over gloo on CPU and compare the result with
the single-process oracle step (which itself is pinned to the reference).
"""

from __future__ import annotations

import numpy as np
import torch

from .pipeline import (F64, SPLAT_KEYS, Cam, adam_update, bin_tiles, cull, decode,
                       flatten_decoded, project, raster, weight_schedule)


def _pack(P: dict) -> torch.Tensor:
    """13 record columns in the CUDA gradient order: mean2d, conic, opacity, color, normal, d."""
    return torch.cat([P["mean2d"], P["conic"], P["opacity"].unsqueeze(-1), P["color"],
                      P["normal_cam"], P["plane_d"].unsqueeze(-1)], dim=-1)


def _unpack(rec: torch.Tensor) -> dict:
    return {"mean2d": rec[:, 0:2], "conic": rec[:, 2:5], "opacity": rec[:, 5],
            "color": rec[:, 6:9], "normal_cam": rec[:, 9:12], "plane_d": rec[:, 12]}


class OracleShardBackend:
    def __init__(self, st, rank: int, world: int, normal_weight: float = 0.0):
        self.st, self.rank, self.world = st, rank, world
        self.normal_weight = float(normal_weight)
        levels = np.asarray(st.levels)
        idx_in_level = np.zeros(levels.shape[0], dtype=np.int64)
        for k in np.unique(levels):
            sel = np.flatnonzero(levels == k)
            idx_in_level[sel] = np.arange(sel.size)
        self.owned = (idx_in_level % world) == rank      # partition.py:49

    def leaves(self):
        st = self.st
        return [*st.weights.values(), st.emb, st.log_scales, st.offsets]

    def schedule(self):
        st = self.st
        w2, w3 = weight_schedule(st.step, st.total_steps, st.step2_start, st.step3_start)
        return w2, w3, self.normal_weight

    def begin_step(self, views, have=(), have_n=()) -> None:
        for p in self.leaves():
            p.requires_grad_(True)
            p.grad = None
        self.B = len(views)
        self.have, self.have_n = list(have), list(have_n)
        self.hw = np.array([v.height * v.width * 3 for v in views], dtype=np.float64)
        self.sums = torch.zeros((self.B, 5), dtype=F64)
        self.work = {}
        self.gaussians = 0

    def grad_like(self) -> torch.Tensor:
        return torch.zeros((0, 13), dtype=F64)

    def forward_shard(self, v: int, view):
        from paper_2503_23044_b200.dist import SplatPayload
        st = self.st
        cam = Cam.of(view)
        act = np.flatnonzero(cull(st.centers, st.levels, st.lod_count, st.lod_ref, st.lod_bias,
                                  cam) & self.owned)
        at = torch.from_numpy(act)
        dec = flatten_decoded(decode(st.weights, st.centers[act], st.emb[at],
                                     torch.exp(st.log_scales[at]), st.offsets[at], cam.center,
                                     st.lod_ref, 3.0 * st.base_voxel_size, st.n))
        gid = (act[:, None] * st.n + np.arange(st.n)).reshape(-1)
        P = project(dec, gid, cam)
        self.gaussians += dec["means"].shape[0]
        self.work[v] = P
        return SplatPayload(_pack(P).detach(), torch.from_numpy(P["zkey"]),
                            torch.from_numpy(P["radius"]), torch.from_numpy(P["gid"]))

    def render(self, v: int, view, payload, image, prior, nprior) -> torch.Tensor:
        st = self.st
        cam = Cam.of(view)
        w2, _ = weight_schedule(st.step, st.total_steps, st.step2_start, st.step3_start)
        order = np.lexsort((payload.gid.numpy(), payload.z.numpy()))
        leaf = payload.rec[torch.from_numpy(order)].clone().requires_grad_(True)
        S = _unpack(leaf)
        offsets, lists = bin_tiles(S["mean2d"].detach().numpy(), payload.radius.numpy()[order],
                                   cam.width, cam.height)
        img = raster(S, offsets, lists, cam)
        gt = torch.as_tensor(np.asarray(image, np.float64))
        diff = (img["rgb"] - gt).abs().sum()
        obj = diff / (self.B * cam.height * cam.width * 3)
        self.sums[v, 0] += float(diff)
        if v in self.have:      # Eq. 9, mean over the views with a prior
            pd = torch.as_tensor(np.asarray(prior[0], np.float64))
            pv = torch.as_tensor(np.asarray(prior[1], bool))
            mask = (pv & img["valid"]).to(F64)
            cnt = int(mask.sum())
            dd = ((img["depth"] - pd).abs() * mask).sum()
            if cnt:
                obj = obj + (w2 / len(self.have)) * dd / cnt
            self.sums[v, 1] += float(dd)
            self.sums[v, 3] += cnt
        if v in self.have_n:    # normal-prior L1 (pipeline.normal_l1_loss)
            pn = torch.as_tensor(np.asarray(nprior[0], np.float64))
            pnv = torch.as_tensor(np.asarray(nprior[1], bool))
            mask = (pnv & img["valid"]).to(F64)
            cnt = int(mask.sum())
            nd = ((img["normal"] - pn).abs().sum(-1) * mask).sum()
            if cnt:
                obj = obj + (self.normal_weight / len(self.have_n)) * nd / (3.0 * cnt)
            self.sums[v, 2] += float(nd)
            self.sums[v, 4] += cnt
        g = torch.autograd.grad(obj, leaf, allow_unused=True)[0]
        g = torch.zeros_like(leaf) if g is None else g
        merged = torch.empty_like(g)
        merged[torch.from_numpy(order)] = g
        return merged

    def backward_shard(self, v: int, view, grads: torch.Tensor) -> None:
        P = self.work[v]
        if grads.shape[0] == 0:
            return
        torch.autograd.backward([_pack(P)], [grads])

    def decoder_grad(self) -> torch.Tensor:
        ws = list(self.st.weights.values())
        self._dflat = torch.cat([(w.grad if w.grad is not None else torch.zeros_like(w)).reshape(-1)
                                 for w in ws])
        return self._dflat

    def loss_terms(self) -> torch.Tensor:
        return self.sums

    def finish_step(self, losses: torch.Tensor) -> dict:
        st = self.st
        off = 0
        for w in st.weights.values():
            k = w.numel()
            w.grad = self._dflat[off:off + k].reshape(w.shape).clone()
            off += k
        w2, _ = weight_schedule(st.step, st.total_steps, st.step2_start, st.step3_start)
        L = losses.numpy()
        rgb = float(np.mean(L[:, 0] / self.hw))
        cnt, ncnt = L[:, 3], L[:, 4]
        dterm = np.where(cnt > 0, L[:, 1] / np.maximum(cnt, 1), 0.0)
        nterm = np.where(ncnt > 0, L[:, 2] / (3.0 * np.maximum(ncnt, 1)), 0.0)
        depth = float(np.mean(dterm[self.have])) if self.have else 0.0
        normal = float(np.mean(nterm[self.have_n])) if self.have_n else 0.0
        for name, p in st.params().items():
            g = p.grad if p.grad is not None else torch.zeros_like(p)
            m, vv = st.moments[name]
            adam_update(p.data, g, m, vv, st.step, st.lr_for(name), st.beta1, st.beta2)
        st.step += 1
        for p in self.leaves():
            p.requires_grad_(False)
            p.grad = None
        return {"total": rgb + w2 * depth + self.normal_weight * normal, "rgb": rgb,
                "depth": depth, "normal": normal, "gaussians": self.gaussians}

    def decoder_checksum(self) -> torch.Tensor:
        return torch.cat([w.detach().reshape(-1) for w in self.st.weights.values()]).view(
            torch.int64).sum().reshape(1)
