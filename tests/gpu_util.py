"""Helpers shared by the GPU parity tests (build device inputs from oracle arrays)."""

from __future__ import annotations

import numpy as np
import torch

import oracle


def f32r(a) -> np.ndarray:
    """Round to float32 and back: the device and the oracle then see equal inputs."""
    return np.asarray(a, np.float32).astype(np.float64)


def records_from(spl: dict) -> "object":
    """Device Projected built from float64 oracle splat arrays (sorted order)."""
    from paper_2503_23044_b200 import device as D
    g = spl["mean2d"].shape[0]
    rec = torch.zeros((max(g, 1), D.REC_F32), dtype=torch.float32)
    rec.view(torch.float64)[:g, 0:2] = torch.as_tensor(np.asarray(spl["mean2d"], np.float64))
    rec[:g, 4:7] = torch.as_tensor(np.asarray(spl["conic"], np.float32))
    rec[:g, 7] = torch.as_tensor(np.asarray(spl["opacity"], np.float32))
    rec[:g, 8:11] = torch.as_tensor(np.asarray(spl["color"], np.float32))
    rec[:g, 11:14] = torch.as_tensor(np.asarray(spl["normal_cam"], np.float32))
    rec[:g, 14] = torch.as_tensor(np.asarray(spl["plane_d"], np.float32))
    rec[:g, 15] = torch.as_tensor(np.arange(g, dtype=np.int32)).view(torch.float32)
    rad = torch.as_tensor(np.asarray(spl["radius"], np.float64))
    z = torch.as_tensor(np.asarray(spl.get("zkey", np.zeros(g)), np.float64)).view(torch.int64)
    return D.Projected(rec[:g].cuda(), rad.cuda(), z.cuda(),
                       torch.arange(g, dtype=torch.int32).cuda(), g)


def splat_arrays(P: dict) -> dict:
    """Oracle splat dict -> numpy float64 arrays rounded like the device record."""
    out = {"mean2d": np.asarray(P["mean2d"].detach().numpy(), np.float64),
           "radius": np.asarray(P["radius"], np.float64),
           "zkey": np.asarray(P["zkey"], np.float64)}
    for k in ("conic", "opacity", "color", "normal_cam", "plane_d"):
        out[k] = f32r(P[k].detach().numpy())
    return out


def oracle_splats(arr: dict) -> dict:
    return {"mean2d": torch.tensor(arr["mean2d"]),
            **{k: torch.tensor(arr[k]) for k in ("conic", "opacity", "color", "normal_cam",
                                                 "plane_d")}}


def guard_mask(img: dict, cam, margin_alpha=1e-3, margin_denom=1e-3) -> np.ndarray:
    """Pixels whose validity decisions are safely away from the guards."""
    a = img["alpha"].detach().numpy() if torch.is_tensor(img["alpha"]) else img["alpha"]
    den = img["denom"].detach().numpy() if torch.is_tensor(img["denom"]) else img["denom"]
    return (np.abs(a - oracle.pipeline.ALPHA_VALID_MIN) > margin_alpha) & \
           (np.abs(np.abs(den) - oracle.pipeline.DENOM_GUARD) > margin_denom)


def rel_close(a, b, rel, floor) -> tuple[bool, float, int]:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    tol = rel * np.maximum(np.abs(a), np.abs(b)) + floor
    bad = np.abs(a - b) > tol
    worst = float((np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)).max()) \
        if a.size else 0.0
    return (not bad.any()), worst, int(bad.sum())
