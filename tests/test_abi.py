"""CPU suite: the C-ABI library (no GPU needed) — symbols, struct layout, workspace planning, error codes."""
import ctypes as C
import os
import re

import pytest

from paper_2007_08501_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "dr_raster.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/dr_raster.h but not exported"
    assert sorted(_lib.EXPORTED_SYMBOLS) == names


def test_settings_layout_matches_header_and_oracle():
    from oracle.oracle import OrcSettings

    assert C.sizeof(_lib.DrRasterSettings) == 48
    for f in ("blur_radius", "znear", "clip_nonpositive_z", "cull_backfaces"):
        assert getattr(_lib.DrRasterSettings, f).offset == getattr(OrcSettings, f).offset


def test_default_settings_are_reference_defaults():
    L = _lib.load()
    s = _lib.DrRasterSettings()
    L.dr_raster_settings_default(C.byref(s))
    # RasterSettings{} (mesh_raster.hpp:18-23) + Camera{} znear (camera.hpp:26)
    assert (s.image_h, s.image_w, s.faces_per_pixel, s.bin_size) == (64, 64, 1, 16)
    assert s.blur_radius == 1e-4 and s.znear == 0.1
    assert (s.clip_nonpositive_z, s.perspective_correct, s.clip_barycentric_coords, s.cull_backfaces) == (1, 0, 1, 0)


def test_workspace_planning_and_validation():
    L = _lib.load()
    s = _lib.DrRasterSettings()
    L.dr_raster_settings_default(C.byref(s))
    n = L.dr_rasterize_meshes_workspace_bytes(2, 1000, C.byref(s))
    assert n >= 16 * 1000 + 4 * 2 * 16 + 4 * 2 * 16 * 1000
    s.bin_size = 0
    assert 16 * 1000 <= L.dr_rasterize_meshes_workspace_bytes(2, 1000, C.byref(s)) < n
    assert L.dr_rasterize_meshes_workspace_bytes(0, 10, C.byref(s)) == 0  # empty batch
    assert "empty mesh batch" in _lib.last_error()
    s.faces_per_pixel = 0
    assert L.dr_rasterize_meshes_workspace_bytes(1, 10, C.byref(s)) == 0
    assert "faces_per_pixel" in _lib.last_error()


def test_error_codes_without_device():
    L = _lib.load()
    s = _lib.DrRasterSettings()
    L.dr_raster_settings_default(C.byref(s))
    nul = C.c_void_p(0)
    rc = L.dr_rasterize_meshes_fwd(nul, nul, nul, 0, 0, C.byref(s), nul, nul, nul, nul, nul, 0, nul)
    assert rc == _lib.DR_ERR_SHAPE
    rc = L.dr_rasterize_meshes_fwd(nul, nul, nul, 1, 0, C.byref(s), nul, nul, nul, nul, nul, 0, nul)
    assert rc == _lib.DR_ERR_USAGE
    s.image_h = 0
    rc = L.dr_rasterize_meshes_bwd(nul, nul, nul, 1, 0, C.byref(s), nul, nul, nul, nul, nul, nul, nul)
    assert rc == _lib.DR_ERR_RANGE
    assert L.dr_profile_kernel_name(2) == b"k_fine"


def test_python_surface_rejects_cpu_tensors():
    import torch

    from paper_2007_08501_b200 import UsageError, rasterize_meshes

    with pytest.raises(UsageError):
        rasterize_meshes(torch.zeros(1, 3, 3, dtype=torch.float64), [0], [1])


def test_shard_libraries_export_dr_shard_h():
    """include/dr_shard.h: the plan / op-list functions live in libdr_raster_b200.so, the NCCL executor in
    libdr_shard_b200.so (loadable without a GPU)."""
    src = open(os.path.join(ROOT, "include", "dr_shard.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = sorted(set(re.findall(r"\b(dr_[a-z0-9_]+)\s*\(", src)))
    assert names == sorted(_lib.SHARD_PLAN_SYMBOLS + _lib.SHARD_NCCL_SYMBOLS)
    L, LS = _lib.load(), _lib.load_shard()
    for n in _lib.SHARD_PLAN_SYMBOLS:
        assert hasattr(L, n), n
    for n in _lib.SHARD_NCCL_SYMBOLS:
        assert hasattr(LS, n), n
    assert C.sizeof(_lib.DrShardOp) == 40 and C.sizeof(_lib.DrShardBuffers) == 40
