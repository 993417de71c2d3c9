"""CPU suite: the oracle restatement against the reference's known answers and golden vectors.

The golden vectors (tests/golden/*.npz) were produced by the reference library itself
(tests/golden/make_golden.py), so this pins the oracle on any box, with or without /root/reference.
"""
import glob
import os

import numpy as np
import pytest

from paper_2007_08501_b200 import scenes as S
from tests._common import orc_settings

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_point_triangle_dist2_known_values(oracle):
    """test_raster.cpp:11-24"""
    a, b, c = [0, 0], [1, 0], [0, 1]
    assert oracle.point_triangle_dist2([0.25, 0.25], a, b, c) == pytest.approx(-0.0625, rel=1e-12)
    assert oracle.point_triangle_dist2([-0.5, 0.5], a, b, c) == pytest.approx(0.25, rel=1e-12)
    assert oracle.point_triangle_dist2([2, 0], a, b, c) == pytest.approx(1.0, rel=1e-12)
    assert oracle.point_triangle_dist2([0.5, 0], a, b, c) == pytest.approx(0.0, abs=1e-15)
    assert oracle.point_triangle_dist2([0.75, 0.75], a, b, c) == pytest.approx(0.125, rel=1e-12)


def test_degenerate_triangles_non_negative(oracle):
    """test_raster.cpp:26-31"""
    a, b, c = [0, 0], [1, 0], [2, 0]
    assert oracle.point_triangle_dist2([1, 0.5], a, b, c) == pytest.approx(0.25)
    assert oracle.point_triangle_dist2([1, 0], a, b, c) == pytest.approx(0.0)
    assert oracle.point_triangle_dist2([3, 0], a, b, c) == pytest.approx(1.0)


def test_kat_golden_bit_identical(oracle):
    g = np.load(os.path.join(GOLDEN, "kat.npz"))
    a, b, c = g["tri"]
    for p, want in zip(g["pts"], g["dist"]):
        assert oracle.point_triangle_dist2(p, a, b, c) == want
    for p, want in zip(g["deg_pts"], g["deg_dist"]):
        assert oracle.point_triangle_dist2(p, [0, 0], [1, 0], [2, 0]) == want


def test_dist_backward_matches_finite_differences(oracle):
    """test_raster.cpp:33-78 (skip near-ties of the nearest edge)."""
    rng = S.Rng(51)
    checked = 0
    for _ in range(40):
        if checked >= 25:
            break
        a = np.array([rng.normal(), rng.normal()])
        b = np.array([rng.normal(), rng.normal()])
        c = np.array([rng.normal(), rng.normal()])
        p = np.array([rng.normal(), rng.normal()])
        area = (b - a)[0] * (c - a)[1] - (b - a)[1] * (c - a)[0]
        if abs(area) < 0.1:
            continue
        ds = []
        for s0, s1 in ((a, b), (b, c), (c, a)):
            ab = s1 - s0
            t = np.clip(np.dot(p - s0, ab) / np.dot(ab, ab), 0, 1)
            ds.append(float(np.sum((p - (s0 + ab * t)) ** 2)))
        ds.sort()
        if ds[1] - ds[0] < 1e-3:
            continue
        checked += 1
        g = oracle.point_triangle_dist2_backward(p, a, b, c)
        eps = 1e-7
        verts = [a, b, c]
        for vi in range(3):
            for ax in range(2):
                vp = [v.copy() for v in verts]
                vm = [v.copy() for v in verts]
                vp[vi][ax] += eps
                vm[vi][ax] -= eps
                fd = (oracle.point_triangle_dist2(p, *vp) - oracle.point_triangle_dist2(p, *vm)) / (2 * eps)
                an = g[vi, ax]
                assert abs(fd - an) / max(abs(fd), abs(an), 1e-8) <= 1e-4
    assert checked >= 15


def test_barycentric_reconstructs_point(oracle):
    """test_raster.cpp:80-97"""
    rng = S.Rng(53)
    for _ in range(30):
        a = np.array([rng.normal(), rng.normal()])
        b = np.array([rng.normal(), rng.normal()])
        c = np.array([rng.normal(), rng.normal()])
        if abs((b - a)[0] * (c - a)[1] - (b - a)[1] * (c - a)[0]) < 0.05:
            continue
        p = np.array([rng.normal(), rng.normal()])
        w = oracle.barycentric(p, a, b, c)
        assert w.sum() == pytest.approx(1.0, rel=1e-9)
        np.testing.assert_allclose(a * w[0] + b * w[1] + c * w[2], p, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(oracle.barycentric([0, 0], [0, 0], [1, 0], [0, 1]), [1, 0, 0], atol=1e-15)


def test_clamp_barycentric(oracle):
    """test_raster.cpp:99-111"""
    np.testing.assert_allclose(oracle.clamp_barycentric([1.5, -0.25, -0.25]), [1, 0, 0])
    np.testing.assert_allclose(oracle.clamp_barycentric([0.2, 0.3, 0.5]), [0.2, 0.3, 0.5])
    m = oracle.clamp_barycentric([0.8, 0.8, -0.6])
    assert m.sum() == pytest.approx(1.0, rel=1e-12) and m[2] == 0.0
    np.testing.assert_allclose(oracle.clamp_barycentric([-1, -2, -3]), [1 / 3] * 3)


def test_pixel_grid(oracle):
    """test_camera.cpp:10-20: pixel (i,j) centre x=(2j+1)/W-1, y=1-(2i+1)/H."""
    import ctypes as C

    xy = np.empty(2)
    for (h, w, i, j) in ((4, 8, 0, 0), (4, 8, 3, 7), (5, 3, 2, 1)):
        oracle.lib.orc_pixel_center_ndc(h, w, i, j, xy.ctypes.data_as(C.POINTER(C.c_double)))
        assert xy[0] == (2.0 * j + 1.0) / w - 1.0 and xy[1] == 1.0 - (2.0 * i + 1.0) / h


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))), ids=os.path.basename)
def test_oracle_matches_reference_golden(path, oracle):
    g = np.load(path)
    if "face_verts" not in g:
        pytest.skip("not a raster fixture")
    H, W, K, _tile = (int(x) for x in g["settings"])
    cam = S.Camera(znear=float(g["znear"]), perspective=bool(g["perspective"]))
    got = oracle.forward(g["face_verts"], g["first"], g["num"], orc_settings(H, K, float(g["blur"]), cam, W=W))
    for name, x in zip(("p2f", "zbuf", "bary", "dists"), got):
        assert np.array_equal(x, g[name]), name
    if "d_verts" in g:
        grad = oracle.backward(g["face_verts"], g["first"], g["num"], orc_settings(H, K, float(g["blur"]), cam, W=W),
                               got[0], got[2], g["d_zbuf"], g["d_bary"], g["d_dists"])
        meshes = S.Meshes([g["verts"]], [g["faces"]])
        cam_full = S.Camera(rotation=g["camera"][1:10].reshape(3, 3), translation=tuple(g["camera"][10:13]),
                            perspective=bool(g["camera"][0]), focal_length=float(g["camera"][13]),
                            principal_point=tuple(g["camera"][14:16]), ortho_scale=tuple(g["camera"][16:18]),
                            znear=float(g["camera"][18]))
        d = S.scatter_face_grads(meshes, cam_full, grad)
        np.testing.assert_allclose(d, g["d_verts"], rtol=1e-12, atol=1e-12)


def test_golden_inputs_regenerate_bit_exact():
    """The numpy scene/camera restatement reproduces the golden inputs (hence the reference's) bit for bit."""
    g = np.load(os.path.join(GOLDEN, "c1.npz"))
    m = S.ico_sphere(3)
    assert np.array_equal(S.face_verts(m, S.bench_camera()), g["face_verts"])
    assert np.array_equal(m.faces_packed(), g["faces"])
