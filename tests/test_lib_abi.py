"""CPU checks of the native boundary: the library loads and exports the C ABI."""

from __future__ import annotations

import ctypes
import re

import pytest

from conftest import ROOT


def _declared() -> list[str]:
    text = (ROOT / "include" / "vsx_b200.h").read_text()
    return sorted(set(re.findall(r"\b(vsx_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_core_entry_points():
    names = _declared()
    for required in ("vsx_cull", "vsx_decode_fwd", "vsx_decode_bwd", "vsx_project_fwd",
                     "vsx_project_bwd", "vsx_sort_pairs_u64", "vsx_bin_count", "vsx_bin_emit",
                     "vsx_raster_fwd", "vsx_raster_bwd", "vsx_l1_loss", "vsx_depth_loss",
                     "vsx_adam", "vsx_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2503_23044_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.skip("libvsx_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding types every exported symbol it uses
    assert set(_lib.EXPORTED) <= set(_declared())
    typed = _lib.load()
    assert typed.vsx_version() == 1
    assert typed.vsx_sort_ws_bytes(1 << 20) > 8 * (1 << 20)


def test_camera_struct_matches_header_layout():
    from paper_2503_23044_b200.geometry import VsxCamera
    # 9 + 3 + 3 + 4 doubles, 2 int32
    assert ctypes.sizeof(VsxCamera) == 19 * 8 + 8


def test_device_entry_points_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_23044_b200.device import require_cuda
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        require_cuda()
