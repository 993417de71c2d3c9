"""Shared helpers for the parity tests (scene -> boundary inputs, settings, comparisons)."""
from __future__ import annotations

import numpy as np

from paper_2007_08501_b200 import scenes as S


def boundary(meshes: S.Meshes, cam: S.Camera):
    """(face_verts [F,3,3], mesh_to_face_first_idx [N], num_faces_per_mesh [N]) the reference derives."""
    return S.face_verts(meshes, cam), meshes.mesh_to_face_first_idx(), meshes.num_faces_per_mesh()


def orc_settings(H, K, blur, cam: S.Camera, W=None, persp_correct=0, clip=1, cull=0, bin_size=16, cap=0):
    from oracle.oracle import make_settings

    return make_settings(H, W or H, K, blur, znear=cam.znear, clip_nonpositive_z=int(cam.perspective),
                         perspective_correct=persp_correct, clip_barycentric_coords=clip, cull_backfaces=cull,
                         bin_size=bin_size, max_faces_per_bin=cap)


def raster_settings(H, K, blur, cam: S.Camera, W=None, persp_correct=False, clip=True, cull=False, bin_size=16,
                    cap=0):
    from paper_2007_08501_b200 import RasterSettings

    return RasterSettings(image_size=(H, W or H), faces_per_pixel=K, blur_radius=blur, bin_size=bin_size,
                          max_faces_per_bin=cap, perspective_correct=persp_correct, clip_barycentric_coords=clip,
                          cull_backfaces=cull, znear=cam.znear, clip_nonpositive_z=cam.perspective)


def acceptance_scenes(n=100):
    """test_acceptance.cpp:143-183 (criterion 4): 100 scenes, sizes/K/blur/tile/camera cycling."""
    rng = S.Rng(1004)
    sizes, ks, blurs = [32, 64, 128], [1, 10, 50], [0.0, 1e-4]
    for trial in range(n):
        if trial % 10 == 0:
            m = S.ico_sphere(1)
        else:
            b = 1 + rng.uniform_int(2)
            m = S.random_soup(rng, b, 60, 25)
        H = sizes[trial % 3]
        K = ks[(trial // 3) % 3]
        blur = blurs[(trial // 9) % 2]
        tile = 16 if trial % 2 else 8
        persp = trial % 4 < 2
        cam = S.Camera.look_from_distance(3.0, persp, 1.5)
        yield trial, m, cam, H, K, blur, tile


def raster_test_scenes(n=20):
    """test_raster.cpp:127-149: 20 random soups."""
    rng = S.Rng(57)
    for trial in range(n):
        m = S.random_soup(rng, 1 + rng.uniform_int(2), 25, 20)
        H = [32, 64][rng.uniform_int(2)]
        K = [1, 10, 50][rng.uniform_int(3)]
        blur = [0.0, 1e-4][rng.uniform_int(2)]
        tile = 16 if rng.uniform_int(2) == 0 else 8
        persp = rng.uniform_int(2) == 0
        cam = S.Camera.look_from_distance(3.0, True, 1.5) if persp else S.Camera.look_from_distance(3.0, False)
        yield trial, m, cam, H, K, blur, tile


def cotangents(S_: int, seed: int = 1):
    """one Rng stream drawn as grad_zbuf (S), then grad_bary (3S), then grad_dists (S)."""
    rng = S.Rng(seed)
    vals = np.array([rng.normal() for _ in range(5 * S_)])
    return vals[:S_], vals[S_:4 * S_], vals[4 * S_:]


def fast_cotangents(S_: int, seed: int = 1):
    """numpy-seeded cotangents for large sizes (not the reference stream)."""
    g = np.random.default_rng(seed)
    return g.standard_normal(S_), g.standard_normal(3 * S_), g.standard_normal(S_)


def rel_err(a, b, floor=1e-12):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), floor)) if a.size else 0.0


GRAD_RTOL, GRAD_ATOL_SCALE = 1e-4, 1e-8


def grad_close(got, want, what="", rtol=GRAD_RTOL, atol_scale=GRAD_ATOL_SCALE):
    """north_star "face_verts gradients within 1e-4 relative", element by element:
    |got - want| <= rtol * |want| + atol_scale * max|want| (the absolute term only absorbs elements whose
    contributions cancel to below atol_scale of the largest gradient). Returns the worst element's err / bound."""
    got, want = np.asarray(got, np.float64).ravel(), np.asarray(want, np.float64).ravel()
    assert got.shape == want.shape, what
    if not want.size:
        return 0.0
    bound = rtol * np.abs(want) + atol_scale * float(np.abs(want).max())
    ratio = np.abs(got - want) / np.maximum(bound, 1e-300)
    i = int(np.argmax(ratio))
    assert ratio[i] <= 1.0, f"{what}: element {i} got {got[i]!r} want {want[i]!r} (err/bound {ratio[i]:.3g})"
    return float(ratio[i])


def parity_report(**kw):
    """Append one JSON line to $DR_PARITY_REPORT (if set): worst-element margins of a parity check."""
    import json
    import os

    path = os.environ.get("DR_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(kw) + "\n")
