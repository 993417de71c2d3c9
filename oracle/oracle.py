"""TEST INFRASTRUCTURE ONLY: ctypes front-ends for the CPU checkers.

* ``Oracle``  -> oracle/liboracle.so, the plain-C restatement (raster_oracle.c) on the face_verts boundary.
* ``RefLib``  -> oracle/_ref/libdr3d_ref.so, the unmodified reference library + extern "C" shim.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may import this
module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdr3d_ref.so")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class OrcSettings(C.Structure):
    """Same layout as dr_raster_settings (include/dr_raster.h)."""

    _fields_ = [
        ("image_h", C.c_int32), ("image_w", C.c_int32), ("faces_per_pixel", C.c_int32),
        ("bin_size", C.c_int32), ("max_faces_per_bin", C.c_int32), ("_pad", C.c_int32),
        ("blur_radius", C.c_double), ("znear", C.c_double),
        ("clip_nonpositive_z", C.c_uint8), ("perspective_correct", C.c_uint8),
        ("clip_barycentric_coords", C.c_uint8), ("cull_backfaces", C.c_uint8), ("_pad2", C.c_uint8 * 4),
    ]


def make_settings(H, W, K, blur=1e-4, znear=0.1, clip_nonpositive_z=1, perspective_correct=0,
                  clip_barycentric_coords=1, cull_backfaces=0, bin_size=16, max_faces_per_bin=0) -> OrcSettings:
    s = OrcSettings()
    s.image_h, s.image_w, s.faces_per_pixel = H, W, K
    s.bin_size, s.max_faces_per_bin = bin_size, max_faces_per_bin
    s.blur_radius, s.znear = blur, znear
    s.clip_nonpositive_z, s.perspective_correct = clip_nonpositive_z, perspective_correct
    s.clip_barycentric_coords, s.cull_backfaces = clip_barycentric_coords, cull_backfaces
    return s


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.orc_rasterize_fwd.argtypes = [_dp, _i64p, _i64p, C.c_int64, C.c_int64, C.POINTER(OrcSettings),
                                        _i64p, _dp, _dp, _dp]
        L.orc_rasterize_bwd.argtypes = [_dp, _i64p, _i64p, C.c_int64, C.c_int64, C.POINTER(OrcSettings),
                                        _i64p, _dp, _dp, _dp, _dp, _dp]
        L.orc_point_triangle_dist2.argtypes = [_dp] * 4
        L.orc_point_triangle_dist2.restype = C.c_double
        L.orc_barycentric.argtypes = [_dp] * 5
        L.orc_clamp_barycentric.argtypes = [_dp, _dp]
        L.orc_point_triangle_dist2_backward.argtypes = [_dp, _dp, _dp, _dp, C.c_double, _dp]
        L.orc_pixel_center_ndc.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.orc_rasterize_points.argtypes = [_dp, _i64p, _i64p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_double, C.c_double, C.c_int, _i64p, _dp, _dp]
        L.orc_rasterize_points_bwd.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, _i64p, _dp, _dp,
                                               _dp]
        L.orc_silhouette_blend.argtypes = [_i64p, _dp, C.c_int64, C.c_int, C.c_double, _dp]
        L.orc_silhouette_blend_backward.argtypes = [_i64p, _dp, C.c_int64, C.c_int, C.c_double, _dp, _dp]

    def rasterize_points(self, points_ndc, first, num, H, W, K, radius, tile=16, znear=0.1, clip_nonpositive_z=1):
        """point_render.cpp:82-155 on points_ndc [P,3]; tile=0 = rasterize_points_naive."""
        pts = np.ascontiguousarray(points_ndc, np.float64)
        first = np.ascontiguousarray(first, np.int64)
        num = np.ascontiguousarray(num, np.int64)
        N = len(first)
        S = N * H * W * K
        idx, zb, d2 = np.empty(S, np.int64), np.empty(S), np.empty(S)
        rc = self.lib.orc_rasterize_points(_p(pts, _dp), _p(first, _i64p), _p(num, _i64p), N, len(pts), H, W, K, tile,
                                           radius, znear, clip_nonpositive_z, _p(idx, _i64p), _p(zb, _dp), _p(d2, _dp))
        if rc:
            raise RuntimeError(f"orc_rasterize_points rc={rc}")
        shp = (N, H, W, K)
        return idx.reshape(shp), zb.reshape(shp), d2.reshape(shp)

    def rasterize_points_backward(self, points_ndc, idx, g_zbuf, g_dists2):
        pts = np.ascontiguousarray(points_ndc, np.float64)
        idx = np.ascontiguousarray(idx, np.int64)
        gz = np.ascontiguousarray(g_zbuf, np.float64)
        gd = np.ascontiguousarray(g_dists2, np.float64)
        N, H, W, K = idx.shape
        g = np.empty((len(pts), 3))
        self.lib.orc_rasterize_points_bwd(_p(pts, _dp), len(pts), N, H, W, K, _p(idx, _i64p), _p(gz, _dp), _p(gd, _dp),
                                          _p(g, _dp))
        return g

    def silhouette_blend(self, p2f, dists, sigma):
        """shading.cpp:75-91 over fragments [N,H,W,K] -> alpha [N,H,W]."""
        p2f = np.ascontiguousarray(p2f, np.int64)
        di = np.ascontiguousarray(dists, np.float64)
        k = p2f.shape[-1]
        out = np.empty(p2f.shape[:-1], np.float64)
        self.lib.orc_silhouette_blend(_p(p2f, _i64p), _p(di, _dp), p2f.size // k, k, sigma, _p(out, _dp))
        return out

    def silhouette_blend_backward(self, p2f, dists, sigma, d_alpha):
        """shading.cpp:93-121 -> d_dists [N,H,W,K]."""
        p2f = np.ascontiguousarray(p2f, np.int64)
        di = np.ascontiguousarray(dists, np.float64)
        da = np.ascontiguousarray(d_alpha, np.float64)
        k = p2f.shape[-1]
        out = np.empty(p2f.shape, np.float64)
        self.lib.orc_silhouette_blend_backward(_p(p2f, _i64p), _p(di, _dp), p2f.size // k, k, sigma, _p(da, _dp),
                                               _p(out, _dp))
        return out

    def forward(self, face_verts, first, num, s: OrcSettings):
        fv = np.ascontiguousarray(face_verts, dtype=np.float64)
        first = np.ascontiguousarray(first, dtype=np.int64)
        num = np.ascontiguousarray(num, dtype=np.int64)
        N, F = len(first), fv.shape[0]
        S = N * s.image_h * s.image_w * s.faces_per_pixel
        p2f = np.empty(S, np.int64)
        zb = np.empty(S, np.float64)
        ba = np.empty(3 * S, np.float64)
        di = np.empty(S, np.float64)
        rc = self.lib.orc_rasterize_fwd(_p(fv, _dp), _p(first, _i64p), _p(num, _i64p), N, F, C.byref(s),
                                        _p(p2f, _i64p), _p(zb, _dp), _p(ba, _dp), _p(di, _dp))
        if rc:
            raise RuntimeError(f"orc_rasterize_fwd rc={rc}")
        shp = (N, s.image_h, s.image_w, s.faces_per_pixel)
        return p2f.reshape(shp), zb.reshape(shp), ba.reshape(shp + (3,)), di.reshape(shp)

    def backward(self, face_verts, first, num, s: OrcSettings, p2f, bary, d_zbuf, d_bary, d_dists):
        fv = np.ascontiguousarray(face_verts, dtype=np.float64)
        first = np.ascontiguousarray(first, dtype=np.int64)
        num = np.ascontiguousarray(num, dtype=np.int64)
        N, F = len(first), fv.shape[0]
        args = [np.ascontiguousarray(x, dtype=t) for x, t in
                ((p2f, np.int64), (bary, np.float64), (d_zbuf, np.float64), (d_bary, np.float64),
                 (d_dists, np.float64))]
        g = np.empty((F, 3, 3), np.float64)
        rc = self.lib.orc_rasterize_bwd(_p(fv, _dp), _p(first, _i64p), _p(num, _i64p), N, F, C.byref(s),
                                        _p(args[0], _i64p), _p(args[1], _dp), _p(args[2], _dp),
                                        _p(args[3], _dp), _p(args[4], _dp), _p(g, _dp))
        if rc:
            raise RuntimeError(f"orc_rasterize_bwd rc={rc}")
        return g

    def point_triangle_dist2(self, p, a, b, c) -> float:
        arr = [np.asarray(x, np.float64) for x in (p, a, b, c)]
        return self.lib.orc_point_triangle_dist2(*[_p(x, _dp) for x in arr])

    def barycentric(self, p, a, b, c):
        arr = [np.asarray(x, np.float64) for x in (p, a, b, c)]
        w = np.empty(3)
        self.lib.orc_barycentric(*[_p(x, _dp) for x in arr], _p(w, _dp))
        return w

    def clamp_barycentric(self, w):
        w = np.asarray(w, np.float64)
        o = np.empty(3)
        self.lib.orc_clamp_barycentric(_p(w, _dp), _p(o, _dp))
        return o

    def point_triangle_dist2_backward(self, p, a, b, c, d_out=1.0):
        arr = [np.asarray(x, np.float64) for x in (p, a, b, c)]
        g = np.empty(6)
        self.lib.orc_point_triangle_dist2_backward(*[_p(x, _dp) for x in arr], d_out, _p(g, _dp))
        return g.reshape(3, 2)


class RefBatch:
    def __init__(self, lib, handle):
        if not handle:
            raise RuntimeError("reference: " + lib.ref_last_error().decode())
        self.lib, self.h = lib, handle
        sz = np.empty(3, np.int64)
        lib.ref_batch_sizes(self.h, _p(sz, _i64p))
        self.n, self.V, self.F = (int(x) for x in sz)

    def export(self):
        v = np.empty((self.V, 3))
        f = np.empty((self.F, 3), np.int64)
        vc = np.empty(self.n, np.int64)
        fc = np.empty(self.n, np.int64)
        self.lib.ref_batch_export(self.h, _p(v, _dp), _p(f, _i64p), _p(vc, _i64p), _p(fc, _i64p))
        return v, f, vc, fc

    def __del__(self):
        try:
            self.lib.ref_batch_free(self.h)
        except Exception:
            pass


class RefLib:
    """The reference's own CPU implementation (dr::rasterize_meshes & co.)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_num_threads.argtypes = [C.c_int]
        L.ref_num_threads.restype = C.c_int
        for fn in ("ref_batch_from_arrays", "ref_ico_sphere", "ref_cube", "ref_synthetic_batch"):
            getattr(L, fn).restype = C.c_void_p
        L.ref_batch_from_arrays.argtypes = [_dp, _i64p, _i64p, _i64p, C.c_int32]
        L.ref_ico_sphere.argtypes = [C.c_int]
        L.ref_cube.argtypes = [C.c_double, C.c_int]
        L.ref_synthetic_batch.argtypes = [C.c_double, C.c_double, C.c_int, C.c_uint64]
        L.ref_batch_free.argtypes = [C.c_void_p]
        L.ref_batch_sizes.argtypes = [C.c_void_p, _i64p]
        L.ref_batch_export.argtypes = [C.c_void_p, _dp, _i64p, _i64p, _i64p]
        L.ref_world_to_ndc.argtypes = [_dp, _dp, C.c_int64, _dp, _dp, _u8p]
        L.ref_world_to_ndc_backward.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, _dp]
        L.ref_rasterize.argtypes = [C.c_void_p, _dp, _i32p, C.c_double, C.c_int, _i64p, _dp, _dp, _dp]
        L.ref_rasterize_backward.argtypes = [C.c_void_p, _dp, _i32p, C.c_double, C.c_int32, _i64p, _dp, _dp,
                                             _dp, _dp, _dp, _dp, _dp]
        L.ref_rasterize_points.argtypes = [_dp, _i64p, C.c_int32, _dp, _i32p, C.c_double, C.c_int, _i64p, _dp, _dp]
        L.ref_splat_position_backward.argtypes = [_dp, _i64p, C.c_int32, _dp, _i32p, C.c_double, _i64p, _dp, _dp,
                                                  _dp, _dp]
        L.ref_softmax_render.argtypes = [C.c_void_p, _dp, _i32p, C.c_double, _dp, _dp, _dp, _i64p]
        L.ref_softmax_render_backward.argtypes = [C.c_void_p, _dp, _i32p, C.c_double, _dp, _dp, _dp, _dp, _dp]
        L.ref_silhouette_blend.argtypes = [_i64p, _dp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, _dp]
        L.ref_silhouette_blend_backward.argtypes = [_i64p, _dp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                    C.c_double, _dp, _dp]
        L.ref_point_triangle_dist2.argtypes = [_dp] * 4
        L.ref_point_triangle_dist2.restype = C.c_double
        L.ref_barycentric.argtypes = [_dp] * 5
        L.ref_clamp_barycentric.argtypes = [_dp, _dp]
        L.ref_point_triangle_dist2_backward.argtypes = [_dp, _dp, _dp, _dp, C.c_double, _dp]
        L.ref_fit_silhouette.argtypes = [C.c_char_p, _i32p, _dp, _dp, _dp, _dp, C.c_int64, _i64p]
        L.ref_mesh_losses.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_silhouette_iou.argtypes = [_dp, _dp, C.c_int64, C.c_double, _dp, _dp]
        L.ref_packed_to_padded.argtypes = [_dp, _i64p, C.c_int64, C.c_int32, C.c_double, _dp]
        L.ref_padded_to_packed.argtypes = [_dp, C.c_int64, C.c_int64, _i64p, C.c_int32, _dp, _i32p]

    def packed_to_padded(self, packed, offsets, pad):
        """dr::packed_to_padded (batching.hpp:48-60) on rows of 1 or 9 doubles -> [B, max_count, row]."""
        x = np.ascontiguousarray(packed, np.float64)
        row = 1 if x.ndim == 1 else int(np.prod(x.shape[1:]))
        off = np.ascontiguousarray(offsets, np.int64)
        B = len(off) - 1
        M = int(np.max(np.diff(off))) if B else 0
        out = np.empty((B, M, row))
        if self.lib.ref_packed_to_padded(_p(x, _dp), _p(off, _i64p), B, row, pad, _p(out, _dp)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out

    def padded_to_packed(self, padded, counts):
        """dr::padded_to_packed (batching.hpp:62-75) -> (packed [sum(counts), row], item_to_element)."""
        x = np.ascontiguousarray(padded, np.float64)
        B, M = x.shape[:2]
        row = int(np.prod(x.shape[2:])) if x.ndim > 2 else 1
        cnt = np.ascontiguousarray(counts, np.int64)
        out = np.empty((int(cnt.sum()), row))
        ite = np.empty(int(cnt.sum()), np.int32)
        if self.lib.ref_padded_to_packed(_p(x, _dp), B, M, _p(cnt, _i64p), row, _p(out, _dp),
                                         ite.ctypes.data_as(_i32p)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out, ite

    def set_num_threads(self, n: int):
        self.lib.ref_set_num_threads(n)

    def num_threads(self) -> int:
        return self.lib.ref_num_threads()

    # batches
    def batch(self, meshes) -> RefBatch:
        v = np.ascontiguousarray(meshes.verts_packed(), np.float64)
        f = np.ascontiguousarray(meshes.faces_local_packed(), np.int64)
        vc = meshes.num_verts_per_mesh()
        fc = meshes.num_faces_per_mesh()
        return RefBatch(self.lib, self.lib.ref_batch_from_arrays(_p(v, _dp), _p(f, _i64p), _p(vc, _i64p),
                                                                 _p(fc, _i64p), len(meshes)))

    def ico_sphere(self, level):
        return RefBatch(self.lib, self.lib.ref_ico_sphere(level))

    def cube(self, half, n):
        return RefBatch(self.lib, self.lib.ref_cube(half, n))

    def synthetic_batch(self, mean, sigma, b, seed):
        return RefBatch(self.lib, self.lib.ref_synthetic_batch(mean, sigma, b, seed))

    def world_to_ndc(self, cam_packed, pts):
        pts = np.ascontiguousarray(pts, np.float64)
        n = len(pts)
        xy, z, cl = np.empty((n, 2)), np.empty(n), np.empty(n, np.uint8)
        cam = np.ascontiguousarray(cam_packed, np.float64)
        if self.lib.ref_world_to_ndc(_p(cam, _dp), _p(pts, _dp), n, _p(xy, _dp), _p(z, _dp), _p(cl, _u8p)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return xy, z, cl.astype(bool)

    def rasterize(self, batch: RefBatch, cam_packed, H, W, K, blur, tile=16, naive=False):
        cam = np.ascontiguousarray(cam_packed, np.float64)
        si = np.array([H, W, K, tile], np.int32)
        S = batch.n * H * W * K
        p2f, zb, ba, di = np.empty(S, np.int64), np.empty(S), np.empty(3 * S), np.empty(S)
        rc = self.lib.ref_rasterize(batch.h, _p(cam, _dp), _p(si, _i32p), blur, int(naive), _p(p2f, _i64p),
                                    _p(zb, _dp), _p(ba, _dp), _p(di, _dp))
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        shp = (batch.n, H, W, K)
        return p2f.reshape(shp), zb.reshape(shp), ba.reshape(shp + (3,)), di.reshape(shp)

    def rasterize_backward(self, batch: RefBatch, cam_packed, H, W, K, blur, frags, d_zbuf, d_bary, d_dists,
                           tile=16):
        cam = np.ascontiguousarray(cam_packed, np.float64)
        si = np.array([H, W, K, tile], np.int32)
        p2f, zb, ba, di = (np.ascontiguousarray(x) for x in frags)
        dz, db, dd = (np.ascontiguousarray(x, np.float64) for x in (d_zbuf, d_bary, d_dists))
        out = np.empty((batch.V, 3))
        rc = self.lib.ref_rasterize_backward(batch.h, _p(cam, _dp), _p(si, _i32p), blur, batch.n,
                                             _p(p2f, _i64p), _p(zb, _dp), _p(ba, _dp), _p(di, _dp),
                                             _p(dz, _dp), _p(db, _dp), _p(dd, _dp), _p(out, _dp))
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out

    def point_triangle_dist2(self, p, a, b, c) -> float:
        arr = [np.asarray(x, np.float64) for x in (p, a, b, c)]
        return self.lib.ref_point_triangle_dist2(*[_p(x, _dp) for x in arr])

    def softmax_render(self, batch: RefBatch, cam_packed, H, W, K, blur, vert_colors, sigma, gamma, bg=(0, 0, 0),
                       tile=16):
        """grad.cpp:181-193: rasterize_meshes -> interpolate_face_attributes -> softmax_blend -> image [n,H,W,3]."""
        cam = np.ascontiguousarray(cam_packed, np.float64)
        si = np.array([H, W, K, tile], np.int32)
        vc = np.ascontiguousarray(vert_colors, np.float64)
        bl = np.array([sigma, gamma, *bg], np.float64)
        img = np.empty((batch.n, H, W, 3))
        p2f = np.empty((batch.n, H, W, K), np.int64)
        if self.lib.ref_softmax_render(batch.h, _p(cam, _dp), _p(si, _i32p), blur, _p(vc, _dp), _p(bl, _dp),
                                       _p(img, _dp), _p(p2f, _i64p)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return img, p2f

    def softmax_render_backward(self, batch: RefBatch, cam_packed, H, W, K, blur, vert_colors, sigma, gamma, d_image,
                                bg=(0, 0, 0), tile=16):
        """grad.cpp:195-206 vjp: (world d_verts [V,3], d_vert_colors [V,3])."""
        cam = np.ascontiguousarray(cam_packed, np.float64)
        si = np.array([H, W, K, tile], np.int32)
        vc = np.ascontiguousarray(vert_colors, np.float64)
        bl = np.array([sigma, gamma, *bg], np.float64)
        di = np.ascontiguousarray(d_image, np.float64)
        dv, dc = np.empty((batch.V, 3)), np.empty((batch.V, 3))
        if self.lib.ref_softmax_render_backward(batch.h, _p(cam, _dp), _p(si, _i32p), blur, _p(vc, _dp), _p(bl, _dp),
                                                _p(di, _dp), _p(dv, _dp), _p(dc, _dp)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return dv, dc

    def rasterize_points(self, points, counts, cam_packed, H, W, K, radius, tile=16, naive=False):
        """dr::rasterize_points / _naive (point_render.hpp:33-36) on world points [P,3] split by counts."""
        pts = np.ascontiguousarray(points, np.float64)
        counts = np.ascontiguousarray(counts, np.int64)
        cam = np.ascontiguousarray(cam_packed, np.float64)
        si = np.array([H, W, K, tile], np.int32)
        n = len(counts)
        S = n * H * W * K
        idx, zb, d2 = np.empty(S, np.int64), np.empty(S), np.empty(S)
        if self.lib.ref_rasterize_points(_p(pts, _dp), _p(counts, _i64p), n, _p(cam, _dp), _p(si, _i32p), radius,
                                         int(naive), _p(idx, _i64p), _p(zb, _dp), _p(d2, _dp)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        shp = (n, H, W, K)
        return idx.reshape(shp), zb.reshape(shp), d2.reshape(shp)

    def splat_position_backward(self, points, counts, cam_packed, H, W, K, radius, frags, d_alphas, tile=16):
        """dr::splat_position_backward (point_render.hpp:66-68): world-space d_points [P,3]."""
        pts = np.ascontiguousarray(points, np.float64)
        counts = np.ascontiguousarray(counts, np.int64)
        cam = np.ascontiguousarray(cam_packed, np.float64)
        si = np.array([H, W, K, tile], np.int32)
        idx, zb, d2 = (np.ascontiguousarray(x) for x in frags)
        da = np.ascontiguousarray(d_alphas, np.float64)
        out = np.empty((len(pts), 3))
        if self.lib.ref_splat_position_backward(_p(pts, _dp), _p(counts, _i64p), len(counts), _p(cam, _dp),
                                                _p(si, _i32p), radius, _p(idx, _i64p), _p(zb, _dp), _p(d2, _dp),
                                                _p(da, _dp), _p(out, _dp)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out

    def silhouette_blend(self, p2f, dists, sigma):
        """dr::silhouette_blend (shading.hpp:37) over fragments [N,H,W,K] -> alpha [N,H,W]."""
        p2f = np.ascontiguousarray(p2f, np.int64)
        di = np.ascontiguousarray(dists, np.float64)
        n, h, w, k = p2f.shape
        out = np.empty((n, h, w), np.float64)
        if self.lib.ref_silhouette_blend(_p(p2f, _i64p), _p(di, _dp), n, h, w, k, sigma, _p(out, _dp)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out

    def silhouette_blend_backward(self, p2f, dists, sigma, d_alpha):
        """dr::silhouette_blend_backward (shading.hpp:39-41) -> d_dists [N,H,W,K]."""
        p2f = np.ascontiguousarray(p2f, np.int64)
        di = np.ascontiguousarray(dists, np.float64)
        da = np.ascontiguousarray(d_alpha, np.float64)
        n, h, w, k = p2f.shape
        out = np.empty((n, h, w, k), np.float64)
        if self.lib.ref_silhouette_blend_backward(_p(p2f, _i64p), _p(di, _dp), n, h, w, k, sigma, _p(da, _dp),
                                                  _p(out, _dp)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return out

    # fit_silhouette (pipeline.cpp:100-205) and its losses (geometry.cpp:556-682)
    def fit_silhouette(self, cfg):
        """cfg: any object with the FitConfig fields (pipeline.hpp:56-78). Returns (trace [iters,5], final loss,
        fitted verts [V,3])."""
        ci = np.array([cfg.template_level, cfg.num_views, cfg.iterations, cfg.image_size, cfg.faces_per_pixel],
                      np.int32)
        cd = np.array([cfg.target_scale, cfg.step_size, cfg.lambda_laplacian, cfg.lambda_edge, cfg.coarse_blur_radius,
                       cfg.coarse_sigma, cfg.coarse_fraction, cfg.blur_radius, cfg.sigma, cfg.camera_distance,
                       cfg.focal_length], np.float64)
        trace = np.zeros((max(cfg.iterations, 0), 5), np.float64)
        vcap = 10 * 4 ** (max(cfg.template_level, 0) + 1) + 2  # ico_sphere(l): 20 * 4^(l+1) faces
        verts = np.zeros((vcap, 3), np.float64)
        fl = np.zeros(1, np.float64)
        nv = np.zeros(1, np.int64)
        if self.lib.ref_fit_silhouette(cfg.target_spec.encode(), _p(ci, _i32p), _p(cd, _dp), _p(trace, _dp),
                                       _p(fl, _dp), _p(verts, _dp), vcap, _p(nv, _i64p)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return trace, float(fl[0]), verts[: int(nv[0])]

    def mesh_losses(self, batch: RefBatch, n_verts: int):
        """(edge_length_loss mean, laplacian_loss mean, d_edge [V,3], d_lap [V,3]) for d_mean = 1."""
        out = np.zeros(2)
        de = np.zeros((n_verts, 3))
        dl = np.zeros((n_verts, 3))
        if self.lib.ref_mesh_losses(batch.h, _p(out, _dp), _p(de, _dp), _p(dl, _dp)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return float(out[0]), float(out[1]), de, dl

    def silhouette_iou(self, pred, gt, d_loss=1.0):
        p = np.ascontiguousarray(pred, np.float64).reshape(-1)
        g = np.ascontiguousarray(gt, np.float64).reshape(-1)
        loss = np.zeros(1)
        grad = np.zeros_like(p)
        if self.lib.ref_silhouette_iou(_p(p, _dp), _p(g, _dp), p.size, d_loss, _p(loss, _dp), _p(grad, _dp)):
            raise RuntimeError(self.lib.ref_last_error().decode())
        return float(loss[0]), grad
