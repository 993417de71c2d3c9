"""B200-native rasterize_meshes: the hot path of arXiv 2007.08501 (PyTorch3D) re-built for sm_100a.

Public surface (mirrors /root/reference/proj/include/dr/mesh_raster.hpp on the north-star boundary):
    RasterSettings, rasterize_meshes, rasterize_meshes_naive, rasterize_meshes_backward, RasterizeMeshes
    rasterize_silhouette, rasterize_silhouette_backward, RasterizeSilhouette (fused silhouette_blend, shading.cpp)
    rasterize_softmax, rasterize_softmax_backward, RasterizeSoftmax, BlendParams (fused softmax render, grad.cpp)
    rasterize_points, rasterize_points_naive, rasterize_points_backward, PointRasterSettings (point_render.cpp)
    fit_silhouette, FitConfig (pipeline.cpp:100-205 on the GPU path; ``fit``)
Input generators and the host camera transform live in ``scenes``; mesh sharding across GPUs in ``shard``.
"""
from .raster import (  # noqa: F401
    BlendParams,
    CudaError,
    KernelTimer,
    MeshIndexError,
    RangeError,
    RasterError,
    RasterizeMeshes,
    RasterizeSilhouette,
    RasterizeSoftmax,
    RasterSettings,
    ShapeError,
    UsageError,
    WorkspaceError,
    bin_stats,
    launch_count,
    rasterize_meshes,
    rasterize_meshes_backward,
    rasterize_meshes_naive,
    rasterize_silhouette,
    rasterize_silhouette_backward,
    rasterize_softmax,
    rasterize_softmax_backward,
    face_verts_backward,
    workspace_bytes,
    world_to_face_verts,
)
from .points import (  # noqa: F401
    PointRasterSettings,
    points_ndc_backward,
    rasterize_points,
    rasterize_points_backward,
    rasterize_points_naive,
    splat_opacity,
    splat_position_backward,
    world_to_points_ndc,
)
from .fit import FitConfig, FitResult, FitTraceRow, NonFiniteError, fit_silhouette  # noqa: F401,E402
