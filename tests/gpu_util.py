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


def adam_worst_bound(lr: float, steps: int) -> float:
    """Largest gap two Adam trajectories (beta1 0.9, beta2 0.999, same start)
    can open in ``steps`` steps: each bias-corrected step moves a parameter
    by at most ~1.5 lr (exactly lr at step 1; |m_hat / sqrt(v_hat)| stays
    below 1.5 for these betas), so 2 x 1.5 lr per step. Post-step parameter
    tests bound their worst element by this, on top of the element-wise check:
    an element whose gradient sits at the float32 noise floor may take an
    Adam step of the other sign, but never more than this."""
    return 3.0 * lr * steps


def noise_floor_close(got, ref, rel, noise) -> tuple[bool, float, int]:
    """Relative closeness with a noise-floor exclusion instead of an allowance.

    An element is left out only when |ref| < noise * rms(ref) of its tensor
    (a gradient whose fp32 sum has no determined sign there); every other
    element must satisfy |got - ref| <= rel * |ref|, and an exactly-zero
    reference (no contribution at all) must be matched by an exact zero.
    Returns (ok, worst relative error over the kept elements, number of
    non-zero elements excluded).
    """
    got, ref = np.asarray(got, np.float64).ravel(), np.asarray(ref, np.float64).ravel()
    if ref.size == 0:
        return True, 0.0, 0
    rms = float(np.sqrt(np.mean(ref * ref)))
    zero = ref == 0.0
    zeros_ok = bool(np.all(got[zero] == 0.0))
    if rms == 0.0:
        return zeros_ok, float(np.abs(got).max()), 0
    keep = np.abs(ref) >= noise * rms
    err = np.abs(got - ref)[keep] / np.abs(ref)[keep]
    worst = float(err.max()) if err.size else 0.0
    return worst <= rel and zeros_ok, worst, int((~keep & ~zero).sum())


def conditioned_close(got, ref, ref_pert, rel, k, eps=0.0) -> tuple[bool, float, float, int]:
    """Element-wise |got - ref| <= rel |ref| + k |ref - ref_pert| + eps rms(ref).

    Nothing is excluded. ``ref_pert`` is the float64 reference evaluated with
    every input (or intermediate) moved by one float32 ulp: |ref - ref_pert|
    is the element's sensitivity to the rounding every float32 evaluation
    carries (a cancelling sum has a large one). ``eps`` rms(ref) is the
    absolute noise floor of float32 accumulation at the tensor's scale.
    Returns (ok, worst err / bound, worst plain relative error over the
    elements whose floors are below rel |ref| / 10, number of elements whose
    floor terms dominate the bound).
    """
    got, ref = np.asarray(got, np.float64).ravel(), np.asarray(ref, np.float64).ravel()
    rms = float(np.sqrt(np.mean(ref * ref))) if ref.size else 0.0
    floor = k * np.abs(ref - np.asarray(ref_pert, np.float64).ravel()) + eps * rms
    err = np.abs(got - ref)
    bound = rel * np.abs(ref) + floor
    zero = bound == 0.0
    ok = bool(np.all(err[zero] == 0.0)) and bool(np.all(err[~zero] <= bound[~zero]))
    ratio = float((err[~zero] / bound[~zero]).max()) if (~zero).any() else 0.0
    well = (floor < 0.1 * rel * np.abs(ref)) & ~zero
    wrel = float((err[well] / np.abs(ref[well])).max()) if well.any() else 0.0
    return ok, ratio, wrel, int((floor > rel * np.abs(ref)).sum())
