"""ctypes binding of libvsx_b200.so (the C ABI in include/vsx_b200.h).

The library is built in-tree (``make -C paper_2503_23044_b200/csrc``) and
loaded from the package directory. There is no fallback: if the shared
object is missing or CUDA is unavailable, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import raise_for_status
from .geometry import VsxCamera

# VSX_LIB points at an alternative build of the same library (A/B timing of
# compile-time variants, scripts/ab_build.sh); the default is the in-tree one.
LIB_PATH = Path(os.environ.get("VSX_LIB") or Path(__file__).resolve().parent / "libvsx_b200.so")

c_void_p = ctypes.c_void_p
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f32 = ctypes.c_float
c_f64 = ctypes.c_double
c_size = ctypes.c_size_t


class VsxDecoder(ctypes.Structure):
    _fields_ = [("w1", c_void_p * 3), ("b1", c_void_p * 3), ("w2", c_void_p * 3),
                ("b2", c_void_p * 3), ("n", c_i32)]


class VsxDecoderGrads(ctypes.Structure):
    _fields_ = [("w1", c_void_p * 3), ("b1", c_void_p * 3), ("w2", c_void_p * 3),
                ("b2", c_void_p * 3)]


class VsxLossDesc(ctypes.Structure):
    """Mirror of vsx_loss_desc (fused RGB-D-N objective of one view)."""

    _fields_ = [("gt_rgb", c_void_p), ("prior_depth", c_void_p),
                ("prior_depth_valid", c_void_p), ("prior_normal", c_void_p),
                ("prior_normal_valid", c_void_p), ("rgb_scale", c_f32),
                ("depth_weight", c_f32), ("normal_weight", c_f32), ("sums", c_void_p),
                ("counts", c_void_p), ("extra_rgb", c_void_p), ("extra_normal", c_void_p),
                ("extra_depth", c_void_p), ("live_pairs", c_void_p),
                ("tile_order", c_void_p), ("sum_partials", c_void_p), ("isect_grad", c_void_p),
                ("tile_live", c_void_p), ("tile_row0", c_i32), ("tile_rows", c_i32)]


class VsxNccGeom(ctypes.Structure):
    """Mirror of vsx_ncc_geom (relative pose + both intrinsics of a view pair)."""

    _fields_ = [("r_rel", c_f64 * 9), ("t_rel", c_f64 * 3),
                ("src_fx", c_f64), ("src_fy", c_f64), ("src_cx", c_f64), ("src_cy", c_f64),
                ("ref_fx", c_f64), ("ref_fy", c_f64), ("ref_cx", c_f64), ("ref_cy", c_f64)]


P = c_void_p
_SIGS = {
    "vsx_version": ([], c_i32),
    "vsx_last_error": ([], ctypes.c_char_p),
    "vsx_sort_ws_bytes": ([c_i64], c_size),
    "vsx_scan_ws_bytes": ([c_i64], c_size),
    "vsx_scan_u32": ([P, P, c_i64, P, c_size, P], c_i32),
    "vsx_sort_pairs_u64": ([P, P, P, P, c_i64, c_i32, c_i32, c_i32, P, c_size, P], c_i32),
    "vsx_sort_pairs_u32": ([P, P, P, P, c_i64, c_i32, c_i32, c_i32, P, c_size, P], c_i32),
    "vsx_tile_ranges": ([P, c_i64, c_i32, P, P], c_i32),
    "vsx_tile_max_len": ([P, c_i32, P, P], c_i32),
    "vsx_sort_splats_ws_bytes": ([c_i64], c_size),
    "vsx_sort_splats_z": ([P, c_i64, P, P, c_size, P], c_i32),
    "vsx_sort_z_gid_ws_bytes": ([c_i64], c_size),
    "vsx_sort_z_gid": ([P, P, P, c_i64, P, c_size, P], c_i32),
    "vsx_select": ([P, c_i64, P, P, P, c_size, P], c_i32),
    "vsx_cull": ([P, P, c_i64, c_i32, c_f64, c_i32, VsxCamera, P, P], c_i32),
    "vsx_decode_fwd": ([VsxDecoder, P, c_i32, P, P, P, P, VsxCamera, c_f64, c_f64,
                        P, P, P, P, P, P, P, P, P, P], c_i32),
    "vsx_decode_bwd_ws_bytes": ([c_i32, c_i32], c_size),
    "vsx_decode_bwd": ([VsxDecoder, VsxDecoderGrads, P, c_i32, P, P, P, P, VsxCamera, c_f64,
                        c_f64, P, P, P, P, P, P, P, P, P, P, P, P, P, P, c_size, P], c_i32),
    "vsx_project_fwd": ([P, P, P, P, P, P, c_i32, VsxCamera, P, P, P, P, P, P], c_i32),
    "vsx_gather_splats": ([P, P, P, c_i32, P, P, P], c_i32),
    "vsx_scatter_rows_f32": ([P, P, c_i32, c_i32, P, P], c_i32),
    "vsx_payload_keys": ([P, P, P, c_i32, c_i32, P, P, P], c_i32),
    "vsx_pack_splat_rows": ([P, P, P, P, c_i32, P, P], c_i32),
    "vsx_splat_rows_keys": ([P, P, c_i32, P, P, P], c_i32),
    "vsx_gather_splat_rows": ([P, P, P, c_i32, P, P, P], c_i32),
    "vsx_bin_count": ([P, P, c_i32, c_i32, c_i32, P, P, P], c_i32),
    "vsx_bin_emit": ([P, P, c_i32, c_i32, c_i32, P, P, P, P], c_i32),
    "vsx_bin_emit_hist": ([P, P, c_i32, c_i32, c_i32, P, P, P, P, P], c_i32),
    "vsx_sort_hist_offset": ([c_i64], ctypes.c_size_t),
    "vsx_raster_fwd": ([P, P, P, VsxCamera, P, P, P, P, P, P, P, P, P], c_i32),
    "vsx_raster_bwd": ([P, P, P, VsxCamera, P, P, P, P, P, P, P, P, P, P, P, P, P], c_i32),
    "vsx_project_bwd": ([P, P, P, P, P, P, c_i32, VsxCamera, P, P, P, P, P, P, P], c_i32),
    "vsx_project_bwd_batch": ([P, P, P, P, P, P, c_i32, c_i32, VsxCamera, P, P, P, P, P, P, P, P,
                               P], c_i32),
    "vsx_l1_loss": ([P, P, c_i64, c_f32, P, P, P], c_i32),
    "vsx_depth_loss": ([P, P, P, P, c_i64, P, P, P, P, P], c_i32),
    "vsx_adam": ([P, P, P, P, c_i32, P, P, c_f64, c_f64, c_f64, c_i32, P], c_i32),
    "vsx_growth_accumulate": ([P, P, c_i32, c_i32, P, P, P], c_i32),
    "vsx_adam_guarded": ([P, P, P, P, c_i32, P, P, c_f64, c_f64, c_f64, c_i32, P, P], c_i32),
    "vsx_masked_l1": ([P, P, P, P, c_i64, c_i32, P, P, P, P, P], c_i32),
    "vsx_launch_count": ([], ctypes.c_uint64),
    "vsx_umma_selftest": ([P, P, P, c_i32, c_i32, c_i32, P], c_i32),
    "vsx_raster_fwd_loss": ([P, P, P, VsxCamera, P, P, P, P, P, P, P, P, VsxLossDesc, P],
                            c_i32),
    "vsx_raster_bwd_loss": ([P, P, P, VsxCamera, P, P, P, P, P, P, P, VsxLossDesc, P, P],
                            c_i32),
    "vsx_decoder_image_floats": ([c_i32], c_size),
    "vsx_decoder_image": ([VsxDecoder, P, P], c_i32),
    "vsx_decode_fwd_tc": ([VsxDecoder, P, P, c_i32, P, P, P, P, VsxCamera, c_f64, c_f64,
                           P, P, P, P, P, P, P, P, P, P], c_i32),
    "vsx_prior_sample": ([P, c_i64, VsxCamera, P, P, P, P, P, P], c_i32),
    "vsx_apply_scale_shift": ([P, P, c_i64, c_f64, c_f64, P, P, P], c_i32),
    "vsx_reprojection_error": ([P, P, VsxCamera, P, P, VsxCamera, P, c_i32, P], c_i32),
    "vsx_enhance_finalize": ([P, P, P, c_f64, c_i64, P, P, P], c_i32),
    "vsx_ncc_patches": ([P, P, P, c_i32, c_i32, P, c_i32, c_i32, VsxNccGeom, P, c_i32, c_i32,
                         P, P, P, P, P, P, P, P, P], c_i32),
    "vsx_ncc_scatter": ([P, c_i32, c_i32, c_i32, P, P, P, P, P, P, c_f64, P, P, P, P], c_i32),
    "vsx_tsdf_integrate": ([P, P, P, P, c_f64, c_f64, P, P, VsxCamera, P, P], c_i32),
    "vsx_bin_emit_tiles": ([P, P, c_i32, c_i32, c_i32, P, P, P, P], c_i32),
    "vsx_tile_segsort": ([P, c_i32, P, c_i32, P], c_i32),
    "vsx_reduce_partials": ([P, c_i64, P, P], c_i32),
    "vsx_raster_grad_reduce": ([P, P, c_i32, c_i32, c_i32, P, P, P, P, P, P], c_i32),
    "vsx_bin_plan_ws_bytes": ([c_i32, c_i32, c_i32], c_size),
    "vsx_bin_build_ws_bytes": ([c_i32, c_i32, c_i64], c_size),
    "vsx_bin_plan": ([P, P, c_i32, c_i32, c_i32, P, c_size, P, P], c_i32),
    "vsx_bin_build": ([c_i32, c_i32, c_i32, c_i64, c_i64, P, c_size, P, c_size, P, P, P], c_i32),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} not built: run `make -C paper_2503_23044_b200/csrc` "
                          "(or __graft_entry__.build())")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke an entry point and raise the mapped exception on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise_for_status(rc, name, lib.vsx_last_error().decode(errors="replace"))


def ptr(t):
    """Device pointer of a tensor as a plain int (None -> NULL): ctypes
    converts ints for c_void_p arguments and struct fields faster than
    c_void_p objects (a call passes up to 20 of them)."""
    return None if t is None else t.data_ptr()


def raw_stream() -> int:
    """cudaStream_t of torch's current stream (the C calls, without the
    Python-level device lookup of torch.cuda.current_stream(): ~15 us per call
    on the host, which a many-view step pays several times per view)."""
    import torch
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def stream() -> c_void_p:
    return c_void_p(raw_stream())
