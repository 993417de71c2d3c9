"""Small invocations of every kernel family, for compute-sanitizer (tools/sanitize.sh).

Each case runs once on a small scene (the sanitizers slow kernels down 10-1000x); correctness is the parity
suites' job, this only has to execute every kernel and code path: the mesh forward (register top-K K <= 8 and
shared-memory lists K > 8, binned / naive / spilled bins, fp32 and fp64 payload), the backward (fp32 / fp64),
the fused silhouette (lane-per-slot kernel K <= 64, lane-per-pixel kernel K > 64) and softmax render (K <= 16
per-pixel, K > 16 slot-compacted), the point rasterizer and its backward, the camera projection / scatter, and
packed <-> padded.

  python tools/sanitize_cases.py [case ...]        (default: all)
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2007_08501_b200 import scenes as S  # noqa: E402

dev = torch.device("cuda:0")
D = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731


def rs(H, K, blur, cam, **kw):
    from paper_2007_08501_b200 import RasterSettings

    return RasterSettings(image_size=H, faces_per_pixel=K, blur_radius=blur, znear=cam.znear,
                          clip_nonpositive_z=cam.perspective, **kw)


def tie_scene(seed):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tests.test_gpu_stress import _tie_scene

    return _tie_scene(seed)


def mesh_case(m, cam, H, K, blur, **kw):
    from paper_2007_08501_b200 import rasterize_meshes, rasterize_meshes_backward

    fv = S.face_verts(m, cam)
    first, num = m.mesh_to_face_first_idx(), m.num_faces_per_mesh()
    s = rs(H, K, blur, cam, **kw)
    for dt in (torch.float32, torch.float64):
        p2f, z, b, d = rasterize_meshes(D(fv), D(first), D(num), s, out_dtype=dt)
        g = torch.Generator(device=dev)
        g.manual_seed(1)
        cot = [torch.randn(t.shape, generator=g, device=dev, dtype=dt) for t in (z, b, d)]
        rasterize_meshes_backward(D(fv), D(first), D(num), s, p2f, b, *cot)
    torch.cuda.synchronize()


def case_mesh():
    cam = S.bench_camera()
    mesh_case(S.ico_sphere(3), cam, 64, 1, 0.0)                                   # C1
    mesh_case(S.ico_sphere(3), cam, 48, 1, 0.0, bin_size=0)                       # naive
    c2 = S.synthetic_batch(3000.0, 1000.0, 3, 0)
    mesh_case(c2, cam, 64, 8, 1e-4)                                               # C2-like, K=8 register path
    mesh_case(c2, cam, 64, 8, 1e-4, perspective_correct=True, cull_backfaces=True)
    mesh_case(c2, cam, 48, 4, 1e-3, bin_size=8, max_faces_per_bin=7)             # forced spill
    mesh_case(tie_scene(4), S.Camera.look_from_distance(3.0, True, 1.6), 44, 64, 3e-3)  # shared-memory lists
    mesh_case(tie_scene(3), S.Camera.look_from_distance(3.0, True, 1.6), 43, 17, 0.0, clip_barycentric_coords=False)


def case_silhouette():
    from paper_2007_08501_b200 import rasterize_silhouette, rasterize_silhouette_backward

    cam = S.bench_camera()
    m = S.synthetic_batch(3000.0, 1000.0, 2, 1)
    fv, first, num = S.face_verts(m, cam), m.mesh_to_face_first_idx(), m.num_faces_per_mesh()
    for K in (8, 50, 80):
        s = rs(48, K, 9e-4, cam)
        p2f, alpha = rasterize_silhouette(D(fv), D(first), D(num), s, 1e-4)
        da = torch.randn(alpha.shape, device=dev, dtype=alpha.dtype)
        rasterize_silhouette_backward(D(fv), D(first), D(num), s, 1e-4, p2f, da)
    torch.cuda.synchronize()


def case_softmax():
    from paper_2007_08501_b200 import BlendParams, rasterize_softmax, rasterize_softmax_backward

    cam = S.bench_camera()
    m = S.synthetic_batch(3000.0, 1000.0, 2, 2)
    fv, first, num = S.face_verts(m, cam), m.mesh_to_face_first_idx(), m.num_faces_per_mesh()
    vc = np.random.default_rng(3).uniform(0.0, 1.0, (len(m.verts_packed()), 3))
    faces = m.faces_packed()
    bp = BlendParams(sigma=1e-4, gamma=1e-4, background_color=(0.2, 0.4, 0.6), znear=cam.znear, zfar=cam.zfar)
    for K in (8, 20):
        s = rs(40, K, 5e-4, cam)
        p2f, img = rasterize_softmax(D(fv), D(first), D(num), s, bp, D(vc), D(faces))
        rasterize_softmax_backward(D(fv), D(first), D(num), s, bp, D(vc), D(faces), p2f,
                                   torch.randn(img.shape, device=dev, dtype=img.dtype))
    torch.cuda.synchronize()


def case_points():
    from paper_2007_08501_b200 import (PointRasterSettings, rasterize_points, rasterize_points_backward,
                                       world_to_points_ndc)

    cam = S.Camera.look_from_distance(3.0, True, 1.5)
    clouds = S.random_clouds(S.Rng(97), 2, 400)
    pts = np.concatenate(clouds, 0)
    num = np.array([len(c) for c in clouds], np.int64)
    first = np.concatenate([[0], np.cumsum(num)[:-1]]).astype(np.int64)
    ndc = world_to_points_ndc(D(pts), cam)
    for bs, K in ((16, 8), (0, 3), (8, 40)):
        s = PointRasterSettings(image_size=48, points_per_pixel=K, radius=0.1, bin_size=bs, znear=cam.znear,
                                clip_nonpositive_z=cam.perspective)
        idx, z, d2 = rasterize_points(ndc, first, num, s)
        rasterize_points_backward(ndc, first, num, s, idx, torch.randn_like(z), torch.randn_like(d2))
    torch.cuda.synchronize()


def case_camera_batching():
    from paper_2007_08501_b200 import face_verts_backward, world_to_face_verts
    from paper_2007_08501_b200.batching import packed_to_padded, padded_to_packed

    cam = S.bench_camera()
    m = S.synthetic_batch(3000.0, 1000.0, 3, 3)
    v, f = D(m.verts_packed()), D(m.faces_packed())
    fv = world_to_face_verts(v, f, cam)
    face_verts_backward(v, f, cam, torch.randn_like(fv))
    first, num = m.mesh_to_face_first_idx(), m.num_faces_per_mesh()
    pad = packed_to_padded(fv.reshape(len(fv), 9), first, num)
    padded_to_packed(pad, first, num, total=len(fv))
    torch.cuda.synchronize()


CASES = {"mesh": case_mesh, "silhouette": case_silhouette, "softmax": case_softmax, "points": case_points,
         "camera_batching": case_camera_batching}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print(f"case {name} done", flush=True)
