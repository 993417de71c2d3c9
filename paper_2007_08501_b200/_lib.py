"""ctypes binding of libdr_raster_b200.so (include/dr_raster.h).

The shared library is built in-tree by ``make`` (or ``__graft_entry__.build()``). There is no fallback: if
the library is missing, importing the package's compute entry points raises.
"""
from __future__ import annotations

import ctypes as C
import os

# DR_RASTER_LIB overrides the in-tree library (used to A/B build variants; the default is the product build)
LIB_PATH = os.environ.get("DR_RASTER_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                           "libdr_raster_b200.so")

DR_OK, DR_ERR_SHAPE, DR_ERR_INDEX, DR_ERR_RANGE, DR_ERR_CUDA, DR_ERR_OOM, DR_ERR_USAGE = range(7)

# symbols include/dr_raster.h declares (the CPU suite checks the library exports all of them)
EXPORTED_SYMBOLS = (
    "dr_raster_settings_default",
    "dr_rasterize_meshes_workspace_bytes",
    "dr_rasterize_meshes_fwd",
    "dr_rasterize_meshes_fwd_f64",
    "dr_rasterize_meshes_bwd",
    "dr_rasterize_meshes_bwd_f64",
    "dr_rasterize_meshes_fwd_hr",
    "dr_rasterize_meshes_bwd_hr",
    "dr_rasterize_silhouette_fwd",
    "dr_rasterize_silhouette_bwd",
    "dr_rasterize_silhouette_fwd_f64",
    "dr_rasterize_silhouette_bwd_f64",
    "dr_rasterize_silhouette_fwd_f64_hr",
    "dr_rasterize_silhouette_bwd_f64_hr",
    "dr_world_to_face_verts_async",
    "dr_rasterize_softmax_fwd",
    "dr_rasterize_softmax_bwd",
    "dr_point_raster_settings_default",
    "dr_rasterize_points_workspace_bytes",
    "dr_rasterize_points_fwd",
    "dr_rasterize_points_fwd_f64",
    "dr_rasterize_points_bwd",
    "dr_rasterize_points_bwd_f64",
    "dr_world_to_points_ndc",
    "dr_points_ndc_backward",
    "dr_world_to_face_verts",
    "dr_face_verts_backward",
    "dr_packed_to_padded",
    "dr_padded_to_packed",
    "dr_packed_item_to_element",
    "dr_last_error",
    "dr_rasterize_meshes_bin_stats",
    "dr_launch_count",
    "dr_profile_enable",
    "dr_profile_read",
    "dr_profile_kernel_name",
    "dr_selftest_division",
    "dr_host_pipeline_create",
    "dr_host_pipeline_groups",
    "dr_host_pipeline_run",
    "dr_host_pipeline_destroy",
)

# include/dr_shard.h: the plan / op-list half lives in libdr_raster_b200.so, the NCCL executor in libdr_shard_b200.so
SHARD_PLAN_SYMBOLS = ("dr_shard_plan_lpt", "dr_shard_gather_ops")
SHARD_NCCL_SYMBOLS = ("dr_shard_unique_id", "dr_shard_comm_init", "dr_shard_comm_destroy", "dr_shard_gather",
                      "dr_shard_last_error")
SHARD_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdr_shard_b200.so")


class DrShardOp(C.Structure):
    """dr_shard_op (include/dr_shard.h)."""

    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("buffer", C.c_int32), ("mesh", C.c_int32),
                ("src_offset", C.c_int64), ("dst_offset", C.c_int64), ("bytes", C.c_int64)]


class DrShardBuffers(C.Structure):
    """dr_shard_buffers (include/dr_shard.h)."""

    _fields_ = [("pix_to_face", C.c_void_p), ("zbuf", C.c_void_p), ("bary", C.c_void_p), ("dists", C.c_void_p),
                ("grad_face_verts", C.c_void_p)]


_shard_lib = None


def load_shard():
    """libdr_shard_b200.so (NCCL executor of the gather); loads libdr_raster_b200.so first."""
    global _shard_lib
    if _shard_lib is not None:
        return _shard_lib
    load()
    if not os.path.exists(SHARD_LIB_PATH):
        raise RuntimeError(f"{SHARD_LIB_PATH} missing: run `make` (it needs NCCL)")
    L = C.CDLL(SHARD_LIB_PATH)
    _vp = C.c_void_p
    L.dr_shard_unique_id.argtypes = [C.c_char_p]
    L.dr_shard_comm_init.argtypes = [C.c_int32, C.c_int32, C.c_char_p, C.POINTER(_vp)]
    L.dr_shard_comm_destroy.argtypes = [_vp]
    L.dr_shard_gather.argtypes = [_vp, C.c_int32, C.c_int64, _vp, _vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_int32, C.POINTER(DrShardBuffers), C.POINTER(DrShardBuffers), _vp]
    for fn in ("dr_shard_unique_id", "dr_shard_comm_init", "dr_shard_comm_destroy", "dr_shard_gather"):
        getattr(L, fn).restype = C.c_int
    L.dr_shard_last_error.restype = C.c_char_p
    _shard_lib = L
    return L


class DrRasterSettings(C.Structure):
    """dr_raster_settings (include/dr_raster.h)."""

    _fields_ = [
        ("image_h", C.c_int32), ("image_w", C.c_int32), ("faces_per_pixel", C.c_int32),
        ("bin_size", C.c_int32), ("max_faces_per_bin", C.c_int32), ("_reserved0", C.c_int32),
        ("blur_radius", C.c_double), ("znear", C.c_double),
        ("clip_nonpositive_z", C.c_uint8), ("perspective_correct", C.c_uint8),
        ("clip_barycentric_coords", C.c_uint8), ("cull_backfaces", C.c_uint8), ("_reserved1", C.c_uint8 * 4),
    ]


class DrPointRasterSettings(C.Structure):
    """dr_point_raster_settings (include/dr_raster.h) = PointRasterSettings (point_render.hpp:14-19)."""

    _fields_ = [
        ("image_h", C.c_int32), ("image_w", C.c_int32), ("points_per_pixel", C.c_int32), ("bin_size", C.c_int32),
        ("radius", C.c_double), ("znear", C.c_double), ("clip_nonpositive_z", C.c_uint8), ("_reserved", C.c_uint8 * 7),
    ]


class DrBlendParams(C.Structure):
    """dr_blend_params (include/dr_raster.h) = BlendParams (shading.hpp:13-17) + Camera znear/zfar."""

    _fields_ = [("sigma", C.c_double), ("gamma", C.c_double), ("background", C.c_double * 3),
                ("znear", C.c_double), ("zfar", C.c_double)]


class DrCamera(C.Structure):
    """dr_camera (include/dr_raster.h) = dr::Camera (camera.hpp:19-35)."""

    _fields_ = [
        ("perspective", C.c_int32), ("_reserved0", C.c_int32), ("rotation", C.c_double * 9),
        ("translation", C.c_double * 3), ("focal_length", C.c_double), ("principal_point", C.c_double * 2),
        ("ortho_scale", C.c_double * 2), ("znear", C.c_double), ("zfar", C.c_double),
    ]


_vp = C.c_void_p
_lib = None


def load() -> C.CDLL:
    """Load (once) and return the library; raises ImportError when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                          "there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    sp = C.POINTER(DrRasterSettings)
    L.dr_raster_settings_default.argtypes = [sp]
    L.dr_rasterize_meshes_workspace_bytes.argtypes = [C.c_int64, C.c_int64, sp]
    L.dr_rasterize_meshes_workspace_bytes.restype = C.c_size_t
    fwd_args = [_vp, _vp, _vp, C.c_int64, C.c_int64, sp, _vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp]
    L.dr_rasterize_meshes_fwd.argtypes = fwd_args
    L.dr_rasterize_meshes_fwd_f64.argtypes = fwd_args
    bwd_args = [_vp, _vp, _vp, C.c_int64, C.c_int64, sp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.dr_rasterize_meshes_bwd.argtypes = bwd_args
    L.dr_rasterize_meshes_bwd_f64.argtypes = bwd_args
    cp = C.POINTER(DrCamera)
    L.dr_world_to_face_verts.argtypes = [_vp, C.c_int64, _vp, C.c_int64, cp, _vp, _vp]
    L.dr_face_verts_backward.argtypes = [_vp, C.c_int64, _vp, C.c_int64, cp, _vp, _vp, _vp]
    L.dr_world_to_face_verts.restype = C.c_int
    L.dr_face_verts_backward.restype = C.c_int
    L.dr_rasterize_meshes_fwd_hr.argtypes = fwd_args + [_vp, _vp]
    L.dr_rasterize_meshes_bwd_hr.argtypes = bwd_args + [_vp, _vp]
    L.dr_rasterize_meshes_fwd_hr.restype = C.c_int
    L.dr_rasterize_meshes_bwd_hr.restype = C.c_int
    L.dr_packed_to_padded.argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp]
    L.dr_padded_to_packed.argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, C.c_int64, _vp, _vp]
    L.dr_packed_item_to_element.argtypes = [_vp, _vp, C.c_int64, C.c_int64, _vp, _vp]
    for fn in ("dr_packed_to_padded", "dr_padded_to_packed", "dr_packed_item_to_element"):
        getattr(L, fn).restype = C.c_int
    L.dr_last_error.restype = C.c_char_p
    L.dr_rasterize_meshes_bin_stats.argtypes = [C.c_int64, C.c_int64, sp, _vp, _vp, C.POINTER(C.c_int64)]
    L.dr_launch_count.restype = C.c_uint64
    L.dr_profile_enable.argtypes = [C.c_int]
    L.dr_profile_read.argtypes = [C.POINTER(C.c_int), C.POINTER(C.c_float), C.c_int]
    L.dr_profile_kernel_name.argtypes = [C.c_int]
    L.dr_profile_kernel_name.restype = C.c_char_p
    for fn in ("dr_rasterize_silhouette_fwd", "dr_rasterize_silhouette_fwd_f64"):
        getattr(L, fn).argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, sp, C.c_double, _vp, _vp, _vp, C.c_size_t, _vp]
    for fn in ("dr_rasterize_silhouette_bwd", "dr_rasterize_silhouette_bwd_f64"):
        getattr(L, fn).argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, sp, C.c_double, _vp, _vp, _vp, _vp]
    L.dr_rasterize_silhouette_fwd_f64_hr.argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, sp, C.c_double, _vp, _vp,
                                                     _vp, C.c_size_t, _vp, _vp, _vp]
    L.dr_rasterize_silhouette_bwd_f64_hr.argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, sp, C.c_double, _vp, _vp,
                                                     _vp, _vp, _vp, _vp]
    L.dr_world_to_face_verts_async.argtypes = [_vp, C.c_int64, _vp, C.c_int64, C.POINTER(DrCamera), _vp, _vp, _vp]
    L.dr_selftest_division.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
    L.dr_selftest_division.restype = C.c_int
    bpp = C.POINTER(DrBlendParams)
    L.dr_rasterize_softmax_fwd.argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, sp, bpp, _vp, _vp, C.c_int64, _vp, _vp,
                                           _vp, C.c_size_t, _vp]
    L.dr_rasterize_softmax_bwd.argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, sp, bpp, _vp, _vp, C.c_int64, _vp, _vp,
                                           _vp, _vp, _vp]
    L.dr_rasterize_softmax_fwd.restype = C.c_int
    L.dr_rasterize_softmax_bwd.restype = C.c_int
    pp = C.POINTER(DrPointRasterSettings)
    L.dr_point_raster_settings_default.argtypes = [pp]
    L.dr_rasterize_points_workspace_bytes.argtypes = [C.c_int64, C.c_int64, pp]
    L.dr_rasterize_points_workspace_bytes.restype = C.c_size_t
    for fn in ("dr_rasterize_points_fwd", "dr_rasterize_points_fwd_f64"):
        getattr(L, fn).argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, pp, _vp, _vp, _vp, _vp, C.c_size_t, _vp]
    for fn in ("dr_rasterize_points_bwd", "dr_rasterize_points_bwd_f64"):
        getattr(L, fn).argtypes = [_vp, _vp, _vp, C.c_int64, C.c_int64, pp, _vp, _vp, _vp, _vp, _vp]
    L.dr_world_to_points_ndc.argtypes = [_vp, C.c_int64, C.POINTER(DrCamera), _vp, _vp]
    L.dr_points_ndc_backward.argtypes = [_vp, C.c_int64, C.POINTER(DrCamera), _vp, _vp, _vp]
    for fn in ("dr_rasterize_points_fwd", "dr_rasterize_points_fwd_f64", "dr_rasterize_points_bwd",
               "dr_rasterize_points_bwd_f64", "dr_world_to_points_ndc", "dr_points_ndc_backward"):
        getattr(L, fn).restype = C.c_int
    for fn in ("dr_rasterize_silhouette_fwd", "dr_rasterize_silhouette_bwd", "dr_rasterize_silhouette_fwd_f64",
               "dr_rasterize_silhouette_bwd_f64", "dr_rasterize_silhouette_fwd_f64_hr",
               "dr_rasterize_silhouette_bwd_f64_hr", "dr_world_to_face_verts_async", "dr_rasterize_meshes_fwd",
               "dr_rasterize_meshes_fwd_f64", "dr_rasterize_meshes_bwd",
               "dr_rasterize_meshes_bwd_f64", "dr_rasterize_meshes_fwd_hr", "dr_rasterize_meshes_bwd_hr",
               "dr_rasterize_meshes_bin_stats"):
        getattr(L, fn).restype = C.c_int
    L.dr_host_pipeline_create.argtypes = [_vp, _vp, C.c_int64, C.c_int64, sp, C.c_int32, C.c_int32, C.c_int32,
                                          C.c_int32, C.POINTER(_vp)]
    L.dr_host_pipeline_groups.argtypes = [_vp, _vp, C.c_int64]
    L.dr_host_pipeline_run.argtypes = [_vp] * 11
    L.dr_host_pipeline_destroy.argtypes = [_vp]
    for fn in ("dr_host_pipeline_create", "dr_host_pipeline_groups", "dr_host_pipeline_run",
               "dr_host_pipeline_destroy"):
        getattr(L, fn).restype = C.c_int
    L.dr_shard_plan_lpt.argtypes = [_vp, C.c_int64, C.c_int32, _vp, _vp]
    L.dr_shard_gather_ops.argtypes = [C.c_int64, _vp, _vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(DrShardOp), C.c_int64,
                                      C.POINTER(C.c_int64)]
    L.dr_shard_plan_lpt.restype = C.c_int
    L.dr_shard_gather_ops.restype = C.c_int
    _lib = L
    return L


def last_error() -> str:
    return load().dr_last_error().decode()
