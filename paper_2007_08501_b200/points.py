"""Point rasterizer on the GPU: rasterize_points / rasterize_points_naive
(/root/reference/proj/include/dr/point_render.hpp:33-36, src/point_render.cpp:82-155) on the points_ndc boundary,
its backward to the projected points, and the camera transform of point clouds.

The reference consumes PointCloudBatch + Camera; like the mesh path the C-ABI consumes what the reference derives:
points_ndc [P,3] f64 = world_to_ndc (x_ndc, y_ndc, z_view) of the packed points (``world_to_points_ndc``) plus
cloud_to_packed_first_idx / num_points_per_cloud. splat_opacity / splat_position_backward (point_render.cpp:157-168,
302-338) are thin compositions on top (``splat_opacity``, ``splat_position_backward``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import torch

from . import _lib
from .raster import RangeError, ShapeError, UsageError, _camera_c, _check, _ptr, _stream


@dataclass
class PointRasterSettings:
    """PointRasterSettings (point_render.hpp:14-19) + the camera fields the boundary needs."""

    image_size: int | tuple = 64
    points_per_pixel: int = 8
    radius: float = 0.05
    bin_size: int = 16           # 0 => rasterize_points_naive; reference `tile_size`
    znear: float = 0.1
    clip_nonpositive_z: bool = True  # perspective camera

    @property
    def hw(self) -> tuple:
        if isinstance(self.image_size, int):
            return (self.image_size, self.image_size)
        return (int(self.image_size[0]), int(self.image_size[1]))

    def to_c(self) -> _lib.DrPointRasterSettings:
        s = _lib.DrPointRasterSettings()
        s.image_h, s.image_w = self.hw
        s.points_per_pixel = int(self.points_per_pixel)
        s.bin_size = int(self.bin_size)
        s.radius = float(self.radius)
        s.znear = float(self.znear)
        s.clip_nonpositive_z = int(bool(self.clip_nonpositive_z))
        return s


def _point_inputs(points_ndc, first, num):
    if not isinstance(points_ndc, torch.Tensor) or not points_ndc.is_cuda:
        raise UsageError("points_ndc must be a CUDA tensor (there is no CPU path)")
    if points_ndc.dim() != 2 or points_ndc.shape[1] != 3:
        raise ShapeError(f"points_ndc must be [P,3], got {tuple(points_ndc.shape)}")
    dev = points_ndc.device
    pts = points_ndc.detach().to(torch.float64).contiguous()
    first = torch.as_tensor(first, dtype=torch.int64, device=dev).contiguous()
    num = torch.as_tensor(num, dtype=torch.int64, device=dev).contiguous()
    if first.dim() != 1 or num.shape != first.shape:
        raise ShapeError("cloud_to_packed_first_idx and num_points_per_cloud must be 1-D of equal length")
    return pts, first, num


def rasterize_points(points_ndc: torch.Tensor, cloud_to_packed_first_idx, num_points_per_cloud,
                     settings: PointRasterSettings | None = None, out_dtype=torch.float32, **kwargs):
    """Returns PointFragments (idx int64 [N,H,W,K], zbuf [N,H,W,K], dists2 [N,H,W,K]) in ``out_dtype``."""
    settings = settings or PointRasterSettings(**kwargs)
    L = _lib.load()
    pts, first, num = _point_inputs(points_ndc, cloud_to_packed_first_idx, num_points_per_cloud)
    N, P = int(first.numel()), int(pts.shape[0])
    H, W = settings.hw
    K = int(settings.points_per_pixel)
    s = settings.to_c()
    dev = pts.device
    ws_n = L.dr_rasterize_points_workspace_bytes(N, P, C.byref(s))
    if ws_n == 0:
        raise (RangeError if N >= 1 else ShapeError)(f"rasterize_points: {_lib.last_error()}")
    if out_dtype not in (torch.float32, torch.float64):
        raise UsageError("out_dtype must be float32 or float64")
    ws = torch.empty(ws_n, dtype=torch.uint8, device=dev)
    idx = torch.empty((N, H, W, K), dtype=torch.int64, device=dev)
    zbuf = torch.empty((N, H, W, K), dtype=out_dtype, device=dev)
    d2 = torch.empty((N, H, W, K), dtype=out_dtype, device=dev)
    fn = L.dr_rasterize_points_fwd if out_dtype == torch.float32 else L.dr_rasterize_points_fwd_f64
    with torch.cuda.device(dev):
        rc = fn(_ptr(pts), _ptr(first), _ptr(num), N, P, C.byref(s), _ptr(idx), _ptr(zbuf), _ptr(d2), _ptr(ws),
                ws.numel(), _stream(dev))
    _check(rc, "rasterize_points")
    return idx, zbuf, d2


def rasterize_points_naive(points_ndc, first, num, settings: PointRasterSettings | None = None,
                           out_dtype=torch.float32, **kwargs):
    """rasterize_points_naive (point_render.hpp:35): every point tested at every pixel (bin_size = 0)."""
    settings = replace(settings or PointRasterSettings(**kwargs), bin_size=0)
    return rasterize_points(points_ndc, first, num, settings, out_dtype=out_dtype)


def rasterize_points_backward(points_ndc, first, num, settings: PointRasterSettings, idx, grad_zbuf, grad_dists2):
    """grad_points_ndc [P,3] f64 from cotangents on zbuf and dists2 (both [N,H,W,K], float32 or float64)."""
    L = _lib.load()
    pts, first, num = _point_inputs(points_ndc, first, num)
    N, P = int(first.numel()), int(pts.shape[0])
    H, W = settings.hw
    shp = (N, H, W, int(settings.points_per_pixel))
    for t in (idx, grad_zbuf, grad_dists2):
        if tuple(t.shape) != shp:
            raise ShapeError(f"rasterize_points_backward: {tuple(t.shape)} does not match fragments {shp}")
    dt = grad_dists2.dtype
    if dt not in (torch.float32, torch.float64):
        raise UsageError("cotangents must be float32 or float64")
    ii = idx.to(torch.int64).contiguous()
    gz, gd = grad_zbuf.to(dt).contiguous(), grad_dists2.to(dt).contiguous()
    grad = torch.zeros((P, 3), dtype=torch.float64, device=pts.device)
    s = settings.to_c()
    fn = L.dr_rasterize_points_bwd if dt == torch.float32 else L.dr_rasterize_points_bwd_f64
    with torch.cuda.device(pts.device):
        rc = fn(_ptr(pts), _ptr(first), _ptr(num), N, P, C.byref(s), _ptr(ii), _ptr(gz), _ptr(gd), _ptr(grad),
                _stream(pts.device))
    _check(rc, "rasterize_points_backward")
    return grad


def world_to_points_ndc(points: torch.Tensor, camera) -> torch.Tensor:
    """world_to_ndc (camera.cpp:36-70) of packed world points [P,3] -> points_ndc [P,3] (bit-identical)."""
    L = _lib.load()
    if not points.is_cuda:
        raise UsageError("points must be a CUDA tensor (there is no CPU path)")
    p = points.detach().to(torch.float64).contiguous()
    out = torch.empty_like(p)
    cam = _camera_c(camera)
    with torch.cuda.device(p.device):
        rc = L.dr_world_to_points_ndc(_ptr(p), p.shape[0], C.byref(cam), _ptr(out), _stream(p.device))
    _check(rc, "world_to_points_ndc")
    return out


def points_ndc_backward(points: torch.Tensor, camera, grad_points_ndc: torch.Tensor) -> torch.Tensor:
    """world_to_ndc_backward (camera.cpp:72-85) per point: grad_points_ndc [P,3] -> world-space grad [P,3]."""
    L = _lib.load()
    p = points.detach().to(torch.float64).contiguous()
    g = grad_points_ndc.to(device=p.device, dtype=torch.float64).contiguous()
    out = torch.empty_like(p)
    cam = _camera_c(camera)
    with torch.cuda.device(p.device):
        rc = L.dr_points_ndc_backward(_ptr(p), p.shape[0], C.byref(cam), _ptr(g), _ptr(out), _stream(p.device))
    _check(rc, "points_ndc_backward")
    return out


def splat_opacity(idx: torch.Tensor, dists2: torch.Tensor, radius: float) -> torch.Tensor:
    """point_render.cpp:157-168: alpha = 1 - dists2 / radius^2 on occupied slots, 0 elsewhere."""
    inv_r2 = 1.0 / (radius * radius)
    return torch.where(idx >= 0, 1.0 - dists2.to(torch.float64) * inv_r2, torch.zeros((), dtype=torch.float64,
                                                                                        device=idx.device))


def splat_position_backward(points: torch.Tensor, camera, points_ndc, first, num, settings: PointRasterSettings, idx,
                            d_alphas: torch.Tensor) -> torch.Tensor:
    """point_render.cpp:302-338: slot alpha cotangents -> world-space d_points [P,3] (through splat_opacity's
    d alpha / d dists2 = -1 / radius^2 and the projection)."""
    inv_r2 = 1.0 / (settings.radius * settings.radius)
    gd = torch.where(idx >= 0, d_alphas.to(torch.float64) * -inv_r2, torch.zeros((), dtype=torch.float64,
                                                                                  device=idx.device))
    g_ndc = rasterize_points_backward(points_ndc, first, num, settings, idx, torch.zeros_like(gd), gd)
    return points_ndc_backward(points, camera, g_ndc)
