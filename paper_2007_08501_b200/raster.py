"""Host-side mirror of the reference operator surface for the rasterize_meshes hot path.

Python over the C-ABI (include/dr_raster.h); PyTorch provides device memory and streams only.

Reference interface this mirrors (/root/reference/proj):
  RasterSettings{image_h, image_w, faces_per_pixel, blur_radius, tile_size}   include/dr/mesh_raster.hpp:18-23
  MeshFragments{pix_to_face, zbuf, bary, dists} as [N,H,W,K(,3)]              include/dr/mesh_raster.hpp:28-39
  rasterize_meshes / rasterize_meshes_naive                                    include/dr/mesh_raster.hpp:41,44
  rasterize_backward (cotangents on zbuf/bary/dists -> vertex grads)            include/dr/mesh_raster.hpp:66-69
  errors: ShapeError / IndexError / RangeError / UsageError                   include/dr/core.hpp:23-49
on the north-star boundary: packed face_verts [F,3,3] (x_ndc, y_ndc, z_view), mesh_to_face_first_idx and
num_faces_per_mesh in; pix_to_face, zbuf, bary_coords, pix_dists out.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib


class RasterError(RuntimeError):
    """Base of the errors the C-ABI reports (dr_status)."""


class ShapeError(RasterError, ValueError):
    """dr::ShapeError (core.hpp:23-25)."""


class MeshIndexError(RasterError, IndexError):
    """dr::IndexError (core.hpp:26-28)."""


class RangeError(RasterError, ValueError):
    """dr::RangeError (core.hpp:38-40)."""


class UsageError(RasterError, ValueError):
    """dr::UsageError (core.hpp:47-49)."""


class CudaError(RasterError):
    pass


class WorkspaceError(RasterError, MemoryError):
    pass


_ERRORS = {
    _lib.DR_ERR_SHAPE: ShapeError,
    _lib.DR_ERR_INDEX: MeshIndexError,
    _lib.DR_ERR_RANGE: RangeError,
    _lib.DR_ERR_CUDA: CudaError,
    _lib.DR_ERR_OOM: WorkspaceError,
    _lib.DR_ERR_USAGE: UsageError,
}


def _check(rc: int, what: str):
    if rc != _lib.DR_OK:
        raise _ERRORS.get(rc, RasterError)(f"{what}: {_lib.last_error()}")


@dataclass
class RasterSettings:
    """RasterSettings (mesh_raster.hpp:18-23) + the north-star parameters + the camera fields the boundary
    needs (znear, clip_nonpositive_z, camera.hpp:26 / camera.cpp:44-47). Defaults are the reference's."""

    image_size: int | tuple = 64
    faces_per_pixel: int = 1
    blur_radius: float = 1e-4
    bin_size: int = 16            # 0 => naive semantics (rasterize_meshes_naive); reference `tile_size`
    max_faces_per_bin: int = 0    # 0 => unlimited (exact-size lists); overflow never changes results
    perspective_correct: bool = False
    clip_barycentric_coords: bool = True
    cull_backfaces: bool = False
    znear: float = 0.1
    clip_nonpositive_z: bool = True  # perspective camera

    @property
    def hw(self) -> tuple:
        if isinstance(self.image_size, int):
            return (self.image_size, self.image_size)
        return (int(self.image_size[0]), int(self.image_size[1]))

    def to_c(self) -> _lib.DrRasterSettings:
        s = _lib.DrRasterSettings()
        s.image_h, s.image_w = self.hw
        s.faces_per_pixel = int(self.faces_per_pixel)
        s.bin_size = int(self.bin_size)
        s.max_faces_per_bin = int(self.max_faces_per_bin)
        s.blur_radius = float(self.blur_radius)
        s.znear = float(self.znear)
        s.clip_nonpositive_z = int(bool(self.clip_nonpositive_z))
        s.perspective_correct = int(bool(self.perspective_correct))
        s.clip_barycentric_coords = int(bool(self.clip_barycentric_coords))
        s.cull_backfaces = int(bool(self.cull_backfaces))
        return s


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _inputs(face_verts, first, num):
    if not isinstance(face_verts, torch.Tensor) or not face_verts.is_cuda:
        raise UsageError("face_verts must be a CUDA tensor (there is no CPU path)")
    if face_verts.dim() != 3 or tuple(face_verts.shape[1:]) != (3, 3):
        raise ShapeError(f"face_verts must be [F,3,3], got {tuple(face_verts.shape)}")
    dev = face_verts.device
    fv = face_verts.detach().to(torch.float64).contiguous()
    first = torch.as_tensor(first, dtype=torch.int64, device=dev).contiguous()
    num = torch.as_tensor(num, dtype=torch.int64, device=dev).contiguous()
    if first.dim() != 1 or num.shape != first.shape:
        raise ShapeError("mesh_to_face_first_idx and num_faces_per_mesh must be 1-D of equal length")
    return fv, first, num


def workspace_bytes(num_meshes: int, num_faces: int, settings: RasterSettings) -> int:
    s = settings.to_c()
    n = _lib.load().dr_rasterize_meshes_workspace_bytes(num_meshes, num_faces, C.byref(s))
    if n == 0:
        raise RangeError(f"invalid settings: {_lib.last_error()}")
    return n


def rasterize_meshes(face_verts: torch.Tensor, mesh_to_face_first_idx, num_faces_per_mesh,
                     settings: RasterSettings | None = None, out_dtype=torch.float32, workspace=None, out=None,
                     host_ranges=None, **kwargs):
    """Forward. Returns (pix_to_face int64 [N,H,W,K], zbuf [N,H,W,K], bary_coords [N,H,W,K,3],
    pix_dists [N,H,W,K]) with zbuf/bary/dists in ``out_dtype`` (float32 or float64). ``out`` = optional
    preallocated (pix_to_face, zbuf, bary_coords, pix_dists), contiguous, written in place. ``host_ranges`` =
    optional (first, num) int64 numpy copies of the mesh ranges: the call then does not synchronise (fp32 only)."""
    settings = settings or RasterSettings(**kwargs)
    L = _lib.load()
    fv, first, num = _inputs(face_verts, mesh_to_face_first_idx, num_faces_per_mesh)
    N, F = int(first.numel()), int(fv.shape[0])
    H, W = settings.hw
    K = int(settings.faces_per_pixel)
    s = settings.to_c()
    dev = fv.device
    ws_n = L.dr_rasterize_meshes_workspace_bytes(N, F, C.byref(s))
    if ws_n == 0:
        _check(_lib.DR_ERR_RANGE if N >= 1 else _lib.DR_ERR_SHAPE, "rasterize_meshes")
    if workspace is None or workspace.numel() < ws_n:
        workspace = torch.empty(ws_n, dtype=torch.uint8, device=dev)
    if out is not None:
        p2f, zbuf, bary, dists = out
        want = [((N, H, W, K), torch.int64), ((N, H, W, K), out_dtype), ((N, H, W, K, 3), out_dtype),
                ((N, H, W, K), out_dtype)]
        for t, (shp, dt) in zip(out, want):
            if tuple(t.shape) != shp or t.dtype != dt or not t.is_contiguous() or t.device != dev:
                raise ShapeError(f"out tensor {tuple(t.shape)} {t.dtype} does not match {shp} {dt}")
    else:
        p2f = torch.empty((N, H, W, K), dtype=torch.int64, device=dev)
        zbuf = torch.empty((N, H, W, K), dtype=out_dtype, device=dev)
        bary = torch.empty((N, H, W, K, 3), dtype=out_dtype, device=dev)
        dists = torch.empty((N, H, W, K), dtype=out_dtype, device=dev)
    fn = L.dr_rasterize_meshes_fwd if out_dtype == torch.float32 else L.dr_rasterize_meshes_fwd_f64
    if out_dtype not in (torch.float32, torch.float64):
        raise UsageError("out_dtype must be float32 or float64")
    with torch.cuda.device(dev):
        if host_ranges is not None and out_dtype == torch.float32:
            hf, hn = (np.ascontiguousarray(x, dtype=np.int64) for x in host_ranges)
            rc = L.dr_rasterize_meshes_fwd_hr(_ptr(fv), _ptr(first), _ptr(num), N, F, C.byref(s), _ptr(p2f),
                                              _ptr(zbuf), _ptr(bary), _ptr(dists), _ptr(workspace), workspace.numel(),
                                              _stream(dev), hf.ctypes.data_as(C.c_void_p),
                                              hn.ctypes.data_as(C.c_void_p))
        else:
            rc = fn(_ptr(fv), _ptr(first), _ptr(num), N, F, C.byref(s), _ptr(p2f), _ptr(zbuf), _ptr(bary),
                    _ptr(dists), _ptr(workspace), workspace.numel(), _stream(dev))
    _check(rc, "rasterize_meshes")
    return p2f, zbuf, bary, dists


def rasterize_meshes_naive(face_verts, mesh_to_face_first_idx, num_faces_per_mesh,
                           settings: RasterSettings | None = None, out_dtype=torch.float32, **kwargs):
    """rasterize_meshes_naive (mesh_raster.hpp:44): the unbinned contract (bin_size = 0)."""
    settings = replace(settings or RasterSettings(**kwargs), bin_size=0)
    return rasterize_meshes(face_verts, mesh_to_face_first_idx, num_faces_per_mesh, settings, out_dtype=out_dtype)


def _host_ranges(host_ranges) -> tuple:
    """(first, num) host copies as contiguous int64 arrays (kept alive by the caller for the call), or ()."""
    if host_ranges is None:
        return ()
    return tuple(np.ascontiguousarray(x, dtype=np.int64) for x in host_ranges)


def _covers(host_ranges, F: int) -> bool:
    """True when the meshes' face ranges cover [0, F) (the backward then overwrites every row of its output)."""
    first, num = (np.asarray(x, dtype=np.int64) for x in host_ranges)
    iv = sorted((int(a), int(a + n)) for a, n in zip(first, num) if n > 0)
    hi = 0
    for a, b in iv:
        if a > hi:
            return False
        hi = max(hi, b)
    return hi >= F


def rasterize_meshes_backward(face_verts, mesh_to_face_first_idx, num_faces_per_mesh, settings: RasterSettings,
                              pix_to_face, bary_coords, grad_zbuf, grad_bary, grad_dists, out=None,
                              host_ranges=None):
    """Backward (rasterize_backward's per-slot part, mesh_raster.cpp:345-378): returns grad_face_verts [F,3,3]
    f64 = d(x_ndc, y_ndc, z_view) per face vertex. Cotangent/bary dtype float32 or float64 (all the same).
    With ``out`` (a contiguous [F,3,3] f64 tensor) only the rows of the batch's face ranges are written."""
    L = _lib.load()
    fv, first, num = _inputs(face_verts, mesh_to_face_first_idx, num_faces_per_mesh)
    N, F = int(first.numel()), int(fv.shape[0])
    H, W = settings.hw
    K = int(settings.faces_per_pixel)
    shp = (N, H, W, K)
    dt = bary_coords.dtype
    if dt not in (torch.float32, torch.float64):
        raise UsageError("bary/cotangents must be float32 or float64")
    tens = [pix_to_face, bary_coords, grad_zbuf, grad_bary, grad_dists]
    want = [shp, shp + (3,), shp, shp + (3,), shp]
    for t, w in zip(tens, want):
        if tuple(t.shape) != w:
            raise ShapeError(f"rasterize_backward: cotangent shapes do not match fragments: {tuple(t.shape)} vs {w}")
    p2f = pix_to_face.to(torch.int64).contiguous()
    others = [t.to(dt).contiguous() for t in tens[1:]]
    if out is not None:
        if tuple(out.shape) != (F, 3, 3) or out.dtype != torch.float64 or not out.is_contiguous():
            raise ShapeError(f"out must be a contiguous [F,3,3] float64 tensor, got {tuple(out.shape)}")
        grad = out
    elif host_ranges is not None and _covers(host_ranges, F):
        grad = torch.empty((F, 3, 3), dtype=torch.float64, device=fv.device)  # every row is overwritten
    else:
        grad = torch.zeros((F, 3, 3), dtype=torch.float64, device=fv.device)
    s = settings.to_c()
    fn = L.dr_rasterize_meshes_bwd if dt == torch.float32 else L.dr_rasterize_meshes_bwd_f64
    with torch.cuda.device(fv.device):
        if host_ranges is not None and dt == torch.float32:
            hf, hn = (np.ascontiguousarray(x, dtype=np.int64) for x in host_ranges)
            rc = L.dr_rasterize_meshes_bwd_hr(_ptr(fv), _ptr(first), _ptr(num), N, F, C.byref(s), _ptr(p2f),
                                              *[_ptr(t) for t in others], _ptr(grad), _stream(fv.device),
                                              hf.ctypes.data_as(C.c_void_p), hn.ctypes.data_as(C.c_void_p))
        else:
            rc = fn(_ptr(fv), _ptr(first), _ptr(num), N, F, C.byref(s), _ptr(p2f), *[_ptr(t) for t in others],
                    _ptr(grad), _stream(fv.device))
    _check(rc, "rasterize_backward")
    return grad


def rasterize_silhouette(face_verts, mesh_to_face_first_idx, num_faces_per_mesh, settings: RasterSettings,
                         sigma: float = 1e-4, want_pix_to_face: bool = True, workspace=None, out_dtype=torch.float32,
                         host_ranges=None):
    """Fused ``silhouette_blend(rasterize_meshes(...), sigma)`` (shading.cpp:75-91 over mesh_raster.cpp:234):
    returns (pix_to_face int64 [N,H,W,K] or None, alpha [N,H,W] in ``out_dtype``, float32 or float64). zbuf /
    bary / dists are never materialised; pix_to_face is what the fused backward needs. ``host_ranges`` =
    (first, num) as host int64 arrays with the device values (float64 only): the call then never synchronises
    (dr_rasterize_silhouette_fwd_f64_hr), e.g. inside a CUDA graph."""
    if out_dtype not in (torch.float32, torch.float64):
        raise UsageError("out_dtype must be float32 or float64")
    if host_ranges is not None and out_dtype != torch.float64:
        raise UsageError("host_ranges needs out_dtype=float64")
    L = _lib.load()
    fv, first, num = _inputs(face_verts, mesh_to_face_first_idx, num_faces_per_mesh)
    N, F = int(first.numel()), int(fv.shape[0])
    H, W = settings.hw
    K = int(settings.faces_per_pixel)
    s = settings.to_c()
    dev = fv.device
    ws_n = L.dr_rasterize_meshes_workspace_bytes(N, F, C.byref(s))
    if ws_n == 0:
        _check(_lib.DR_ERR_RANGE if N >= 1 else _lib.DR_ERR_SHAPE, "rasterize_silhouette")
    if workspace is None or workspace.numel() < ws_n:
        workspace = torch.empty(ws_n, dtype=torch.uint8, device=dev)
    p2f = torch.empty((N, H, W, K), dtype=torch.int64, device=dev) if want_pix_to_face else None
    alpha = torch.empty((N, H, W), dtype=out_dtype, device=dev)
    fn = L.dr_rasterize_silhouette_fwd if out_dtype == torch.float32 else L.dr_rasterize_silhouette_fwd_f64
    hr = _host_ranges(host_ranges)
    if hr:
        fn = L.dr_rasterize_silhouette_fwd_f64_hr
    with torch.cuda.device(dev):
        rc = fn(_ptr(fv), _ptr(first), _ptr(num), N, F, C.byref(s), float(sigma), _ptr(p2f), _ptr(alpha),
                _ptr(workspace), workspace.numel(), _stream(dev), *[a.ctypes.data_as(C.c_void_p) for a in hr])
    _check(rc, "rasterize_silhouette")
    return p2f, alpha


def rasterize_silhouette_backward(face_verts, mesh_to_face_first_idx, num_faces_per_mesh, settings: RasterSettings,
                                  sigma: float, pix_to_face, grad_alpha, host_ranges=None, out=None):
    """Fused ``rasterize_backward(..., 0, 0, silhouette_blend_backward(frag, sigma, grad_alpha))``
    (shading.cpp:93-121 + mesh_raster.cpp:329-403, the reference fit loop pipeline.cpp:153-162): returns
    grad_face_verts [F,3,3] f64 (z components are zero: only the distance envelope carries gradient). A float64
    grad_alpha selects the fp64 entry point (fp64 sigmoid), anything else is read as float32. ``host_ranges``
    (float64 only) makes the call non-synchronising; ``out`` receives grad_face_verts (overwritten on the batch's
    face ranges)."""
    L = _lib.load()
    fv, first, num = _inputs(face_verts, mesh_to_face_first_idx, num_faces_per_mesh)
    N, F = int(first.numel()), int(fv.shape[0])
    H, W = settings.hw
    K = int(settings.faces_per_pixel)
    if tuple(pix_to_face.shape) != (N, H, W, K) or tuple(grad_alpha.shape) != (N, H, W):
        raise ShapeError(f"rasterize_silhouette_backward: pix_to_face {tuple(pix_to_face.shape)} / grad_alpha "
                         f"{tuple(grad_alpha.shape)} do not match [N,H,W,K] / [N,H,W] = {(N, H, W, K)}")
    p2f = pix_to_face.to(torch.int64).contiguous()
    f64 = grad_alpha.dtype == torch.float64
    if host_ranges is not None and not f64:
        raise UsageError("host_ranges needs a float64 grad_alpha")
    ga = grad_alpha.to(torch.float64 if f64 else torch.float32).contiguous()
    grad = out if out is not None else torch.zeros((F, 3, 3), dtype=torch.float64, device=fv.device)
    s = settings.to_c()
    fn = L.dr_rasterize_silhouette_bwd_f64 if f64 else L.dr_rasterize_silhouette_bwd
    hr = _host_ranges(host_ranges)
    if hr:
        fn = L.dr_rasterize_silhouette_bwd_f64_hr
    with torch.cuda.device(fv.device):
        rc = fn(_ptr(fv), _ptr(first), _ptr(num), N, F, C.byref(s), float(sigma), _ptr(p2f), _ptr(ga), _ptr(grad),
                _stream(fv.device), *[a.ctypes.data_as(C.c_void_p) for a in hr])
    _check(rc, "rasterize_silhouette_backward")
    return grad


class RasterizeSilhouette(torch.autograd.Function):
    """Autograd wrapper of the fused silhouette path: face_verts -> alpha [N,H,W]."""

    @staticmethod
    def forward(ctx, face_verts, first, num, settings: RasterSettings, sigma: float):
        p2f, alpha = rasterize_silhouette(face_verts, first, num, settings, sigma)
        ctx.settings, ctx.sigma = settings, sigma
        ctx.save_for_backward(face_verts, torch.as_tensor(first, device=face_verts.device),
                              torch.as_tensor(num, device=face_verts.device), p2f)
        return alpha

    @staticmethod
    def backward(ctx, g_alpha):
        fv, first, num, p2f = ctx.saved_tensors
        g = rasterize_silhouette_backward(fv, first, num, ctx.settings, ctx.sigma, p2f, g_alpha)
        return g.to(fv.dtype), None, None, None, None


@dataclass
class BlendParams:
    """BlendParams (shading.hpp:13-17) + the camera's znear / zfar used by softmax_blend's depth normalisation."""

    sigma: float = 1e-4
    gamma: float = 1e-4
    background_color: tuple = (0.0, 0.0, 0.0)
    znear: float = 0.1
    zfar: float = 100.0

    def to_c(self) -> _lib.DrBlendParams:
        b = _lib.DrBlendParams()
        b.sigma, b.gamma = float(self.sigma), float(self.gamma)
        for i in range(3):
            b.background[i] = float(self.background_color[i])
        b.znear, b.zfar = float(self.znear), float(self.zfar)
        return b


def _blend_inputs(vert_colors, faces, dev):
    vc = torch.as_tensor(vert_colors).to(device=dev, dtype=torch.float64).contiguous()
    fc = torch.as_tensor(faces).to(device=dev, dtype=torch.int64).contiguous()
    if vc.dim() != 2 or vc.shape[1] != 3 or fc.dim() != 2 or fc.shape[1] != 3:
        raise ShapeError(f"vert_colors must be [V,3] and faces [F,3], got {tuple(vc.shape)} / {tuple(fc.shape)}")
    return vc, fc


def rasterize_softmax(face_verts, mesh_to_face_first_idx, num_faces_per_mesh, settings: RasterSettings,
                      blend: BlendParams, vert_colors, faces, want_pix_to_face: bool = True, workspace=None):
    """Fused softmax render (grad.cpp:177-193): rasterize_meshes -> interpolate_face_attributes(vert_colors) ->
    softmax_blend. Returns (pix_to_face int64 [N,H,W,K] or None, image float32 [N,H,W,3])."""
    L = _lib.load()
    fv, first, num = _inputs(face_verts, mesh_to_face_first_idx, num_faces_per_mesh)
    vc, fc = _blend_inputs(vert_colors, faces, fv.device)
    if fc.shape[0] != fv.shape[0]:
        raise ShapeError(f"faces [{fc.shape[0]},3] does not match face_verts [{fv.shape[0]},3,3]")
    N, F = int(first.numel()), int(fv.shape[0])
    H, W = settings.hw
    K = int(settings.faces_per_pixel)
    s = settings.to_c()
    b = blend.to_c()
    dev = fv.device
    ws_n = L.dr_rasterize_meshes_workspace_bytes(N, F, C.byref(s))
    if ws_n == 0:
        _check(_lib.DR_ERR_RANGE if N >= 1 else _lib.DR_ERR_SHAPE, "rasterize_softmax")
    if workspace is None or workspace.numel() < ws_n:
        workspace = torch.empty(ws_n, dtype=torch.uint8, device=dev)
    p2f = torch.empty((N, H, W, K), dtype=torch.int64, device=dev) if want_pix_to_face else None
    image = torch.empty((N, H, W, 3), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        rc = L.dr_rasterize_softmax_fwd(_ptr(fv), _ptr(first), _ptr(num), N, F, C.byref(s), C.byref(b), _ptr(vc),
                                        _ptr(fc), vc.shape[0], _ptr(p2f), _ptr(image), _ptr(workspace),
                                        workspace.numel(), _stream(dev))
    _check(rc, "rasterize_softmax")
    return p2f, image


def rasterize_softmax_backward(face_verts, mesh_to_face_first_idx, num_faces_per_mesh, settings: RasterSettings,
                               blend: BlendParams, vert_colors, faces, pix_to_face, grad_image):
    """vjp of the softmax render (grad.cpp:195-206): returns (grad_face_verts [F,3,3] f64, grad_vert_colors [V,3]
    f64), one fused kernel (dr_rasterize_softmax_bwd)."""
    L = _lib.load()
    fv, first, num = _inputs(face_verts, mesh_to_face_first_idx, num_faces_per_mesh)
    vc, fc = _blend_inputs(vert_colors, faces, fv.device)
    N, F = int(first.numel()), int(fv.shape[0])
    H, W = settings.hw
    K = int(settings.faces_per_pixel)
    if tuple(pix_to_face.shape) != (N, H, W, K) or tuple(grad_image.shape) != (N, H, W, 3):
        raise ShapeError("rasterize_softmax_backward: pix_to_face / grad_image do not match [N,H,W,K] / [N,H,W,3]")
    p2f = pix_to_face.to(torch.int64).contiguous()
    gi = grad_image.to(torch.float32).contiguous()
    g_fv = torch.zeros((F, 3, 3), dtype=torch.float64, device=fv.device)
    g_vc = torch.zeros_like(vc)
    s = settings.to_c()
    b = blend.to_c()
    with torch.cuda.device(fv.device):
        rc = L.dr_rasterize_softmax_bwd(_ptr(fv), _ptr(first), _ptr(num), N, F, C.byref(s), C.byref(b), _ptr(vc),
                                        _ptr(fc), vc.shape[0], _ptr(p2f), _ptr(gi), _ptr(g_fv), _ptr(g_vc),
                                        _stream(fv.device))
    _check(rc, "rasterize_softmax_backward")
    return g_fv, g_vc


class RasterizeSoftmax(torch.autograd.Function):
    """Autograd wrapper of the fused softmax render: (face_verts, vert_colors) -> image [N,H,W,3]."""

    @staticmethod
    def forward(ctx, face_verts, vert_colors, faces, first, num, settings: RasterSettings, blend: BlendParams):
        p2f, image = rasterize_softmax(face_verts, first, num, settings, blend, vert_colors, faces)
        ctx.settings, ctx.blend = settings, blend
        ctx.save_for_backward(face_verts, vert_colors, torch.as_tensor(faces, device=face_verts.device),
                              torch.as_tensor(first, device=face_verts.device),
                              torch.as_tensor(num, device=face_verts.device), p2f)
        return image

    @staticmethod
    def backward(ctx, g_image):
        fv, vc, faces, first, num, p2f = ctx.saved_tensors
        g_fv, g_vc = rasterize_softmax_backward(fv, first, num, ctx.settings, ctx.blend, vc, faces, p2f, g_image)
        return g_fv.to(fv.dtype), g_vc.to(vc.dtype), None, None, None, None, None


def bin_stats(num_meshes, num_faces, settings: RasterSettings, workspace: torch.Tensor) -> dict:
    """Coarse-stage counters left in the workspace by the last forward (synchronises)."""
    L = _lib.load()
    out = (C.c_int64 * 4)()
    s = settings.to_c()
    rc = L.dr_rasterize_meshes_bin_stats(num_meshes, num_faces, C.byref(s), _ptr(workspace),
                                         _stream(workspace.device), out)
    _check(rc, "bin_stats")
    return dict(bins=out[0], overflowed=out[1], entries=out[2], max_bin=out[3])


class RasterizeMeshes(torch.autograd.Function):
    """Autograd wrapper: face_verts -> (pix_to_face, zbuf, bary_coords, pix_dists)."""

    @staticmethod
    def forward(ctx, face_verts, first, num, settings: RasterSettings):
        p2f, zbuf, bary, dists = rasterize_meshes(face_verts, first, num, settings)
        ctx.settings = settings
        ctx.save_for_backward(face_verts, torch.as_tensor(first, device=face_verts.device),
                              torch.as_tensor(num, device=face_verts.device), p2f, bary)
        ctx.mark_non_differentiable(p2f)
        return p2f, zbuf, bary, dists

    @staticmethod
    def backward(ctx, _g_p2f, g_zbuf, g_bary, g_dists):
        fv, first, num, p2f, bary = ctx.saved_tensors
        zeros = lambda t, like: torch.zeros_like(like) if t is None else t  # noqa: E731
        g = rasterize_meshes_backward(fv, first, num, ctx.settings, p2f, bary, zeros(g_zbuf, bary[..., 0]),
                                      zeros(g_bary, bary), zeros(g_dists, bary[..., 0]))
        return g.to(fv.dtype), None, None, None


def _camera_c(cam) -> _lib.DrCamera:
    """scenes.Camera (or any object with the dr::Camera fields) -> dr_camera."""
    c = _lib.DrCamera()
    c.perspective = int(bool(cam.perspective))
    rot = [float(x) for row in cam.rotation for x in row]
    for i in range(9):
        c.rotation[i] = rot[i]
    for i in range(3):
        c.translation[i] = float(cam.translation[i])
    c.focal_length = float(cam.focal_length)
    c.principal_point[0], c.principal_point[1] = (float(x) for x in cam.principal_point)
    c.ortho_scale[0], c.ortho_scale[1] = (float(x) for x in cam.ortho_scale)
    c.znear, c.zfar = float(cam.znear), float(cam.zfar)
    return c


def world_to_face_verts(verts: torch.Tensor, faces: torch.Tensor, camera, check: bool = True,
                        bad_index: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """world_to_ndc (camera.cpp:36-70) + per-face gather on the GPU: verts [V,3] f64 world space, faces [F,3] packed
    global vertex ids -> face_verts [F,3,3] (x_ndc, y_ndc, z_view), bit-identical to the reference."""
    L = _lib.load()
    if not verts.is_cuda:
        raise UsageError("verts must be a CUDA tensor (there is no CPU path)")
    v = verts.detach().to(torch.float64).contiguous()
    f = faces.to(device=v.device, dtype=torch.int64).contiguous()
    if out is None:
        out = torch.empty((f.shape[0], 3, 3), dtype=torch.float64, device=v.device)
    cam = _camera_c(camera)
    with torch.cuda.device(v.device):
        if check:  # validates the vertex indices (one synchronisation)
            rc = L.dr_world_to_face_verts(_ptr(v), v.shape[0], _ptr(f), f.shape[0], C.byref(cam), _ptr(out),
                                          _stream(v.device))
        else:  # no synchronisation (CUDA-graph capturable); bad indices flag `bad_index` (device int32)
            rc = L.dr_world_to_face_verts_async(_ptr(v), v.shape[0], _ptr(f), f.shape[0], C.byref(cam), _ptr(out),
                                                _ptr(bad_index), _stream(v.device))
    _check(rc, "world_to_face_verts")
    return out


def face_verts_backward(verts: torch.Tensor, faces: torch.Tensor, camera, grad_face_verts: torch.Tensor):
    """grad_face_verts [F,3,3] -> world-space grad_verts [V,3] (vertex scatter + world_to_ndc_backward,
    mesh_raster.cpp:380-401, camera.cpp:72-85)."""
    L = _lib.load()
    v = verts.detach().to(torch.float64).contiguous()
    f = faces.to(device=v.device, dtype=torch.int64).contiguous()
    g = grad_face_verts.to(device=v.device, dtype=torch.float64).contiguous()
    out = torch.empty((v.shape[0], 3), dtype=torch.float64, device=v.device)
    cam = _camera_c(camera)
    with torch.cuda.device(v.device):
        rc = L.dr_face_verts_backward(_ptr(v), v.shape[0], _ptr(f), f.shape[0], C.byref(cam), _ptr(g), _ptr(out),
                                      _stream(v.device))
    _check(rc, "face_verts_backward")
    return out


def launch_count() -> int:
    return int(_lib.load().dr_launch_count())


class KernelTimer:
    """Per-kernel CUDA-event timing recorded by the library on the launching stream."""

    def __enter__(self):
        _lib.load().dr_profile_enable(1)
        return self

    def __exit__(self, *exc):
        L = _lib.load()
        cap = 1 << 16
        idx = (C.c_int * cap)()
        ms = (C.c_float * cap)()
        n = L.dr_profile_read(idx, ms, cap)
        self.records = [(L.dr_profile_kernel_name(idx[i]).decode(), ms[i]) for i in range(n)]
        L.dr_profile_enable(0)
        return False

    def total(self, name: str) -> tuple:
        t = [ms for k, ms in self.records if k == name]
        return (sum(t), len(t))
