"""CPU suite: pins the scene generators and the oracle restatement against the REFERENCE LIBRARY itself
(oracle/_ref/libdr3d_ref.so = unmodified /root/reference sources + extern "C" shim). Skipped where the
reference library was not built."""
import math

import numpy as np
import pytest

from paper_2007_08501_b200 import scenes as S
from tests._common import acceptance_scenes, boundary, cotangents, orc_settings, raster_test_scenes


def test_templates_bit_exact(reflib):
    for lvl in range(0, 5):
        v, f, _, _ = reflib.ico_sphere(lvl).export()
        m = S.ico_sphere(lvl)
        assert np.array_equal(m.verts[0], v) and np.array_equal(m.faces[0], f)
    for n in (1, 2, 7, 32):
        v, f, _, _ = reflib.cube(0.8, n).export()
        m = S.cube(0.8, n)
        assert np.array_equal(m.verts[0], v) and np.array_equal(m.faces[0], f)
    v, f, vc, fc = reflib.synthetic_batch(11000.0, 18000.0 / (2 * math.sqrt(3.0)), 8, 0).export()
    m = S.config_meshes("C2")
    assert np.array_equal(m.verts_packed(), v) and np.array_equal(m.faces_packed(), f)
    assert fc.tolist() == [20480, 12288, 3072, 20480, 3072, 6912, 5120, 12288]


def test_world_to_ndc_bit_exact(reflib):
    m = S.config_meshes("C2")
    for cam in (S.bench_camera(), S.Camera.look_from_distance(3.0, False),
                S.Camera(rotation=S.axis_angle((0.3, -1.0, 0.2), 0.7), translation=(0.1, -0.2, 2.5),
                         focal_length=1.7, principal_point=(0.05, -0.02))):
        xy, z, cl = S.world_to_ndc(cam, m.verts_packed())
        xy2, z2, cl2 = reflib.world_to_ndc(cam.packed(), m.verts_packed())
        assert np.array_equal(xy, xy2) and np.array_equal(z, z2) and np.array_equal(cl, cl2)


@pytest.mark.parametrize("which", ["raster", "acceptance"])
def test_oracle_equals_reference_on_reference_scenes(which, reflib, oracle):
    gen = raster_test_scenes(20) if which == "raster" else acceptance_scenes(100)
    for trial, m, cam, H, K, blur, tile in gen:
        want = reflib.rasterize(reflib.batch(m), cam.packed(), H, H, K, blur, tile)
        naive = reflib.rasterize(reflib.batch(m), cam.packed(), H, H, K, blur, tile, naive=True)
        fv, first, num = boundary(m, cam)
        got = oracle.forward(fv, first, num, orc_settings(H, K, blur, cam))
        for x, y, z in zip(got, want, naive):
            assert np.array_equal(x, y) and np.array_equal(y, z), f"{which} trial {trial}"


def test_oracle_equals_reference_c2_forward_backward(reflib, oracle):
    m, cam = S.config_meshes("C2"), S.bench_camera()
    rb = reflib.batch(m)
    want = reflib.rasterize(rb, cam.packed(), 128, 128, 8, 1e-4)
    fv, first, num = boundary(m, cam)
    o = orc_settings(128, 8, 1e-4, cam)
    got = oracle.forward(fv, first, num, o)
    for x, y in zip(got, want):
        assert np.array_equal(x, y)
    assert (got[0] >= 0).sum() == 570472
    dz, db, dd = cotangents(got[0].size)
    d_ref = reflib.rasterize_backward(rb, cam.packed(), 128, 128, 8, 1e-4, want, dz, db, dd)
    g = oracle.backward(fv, first, num, o, got[0], got[2], dz, db, dd)
    d = S.scatter_face_grads(m, cam, g)
    assert np.max(np.abs(d - d_ref)) <= 1e-12 * np.max(np.abs(d_ref))


def test_backface_sign_convention(reflib):
    """cull_backfaces culls NDC signed_area2 > 0: on an outward-wound closed mesh the camera-facing faces
    have negative NDC area; check that culling keeps exactly the visible surface."""
    m = S.ico_sphere(3)
    for cam in (S.bench_camera(), S.Camera.look_from_distance(3.0, False)):
        fv = S.face_verts(m, cam)
        a, b, c = fv[:, 0, :2], fv[:, 1, :2], fv[:, 2, :2]
        area = (b - a)[:, 0] * (c - a)[:, 1] - (b - a)[:, 1] * (c - a)[:, 0]
        tri = m.verts[0][m.faces[0]]
        normal = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])  # outward (CCW seen from outside)
        view = S.world_to_view(cam, tri[:, 0])
        facing = np.einsum("ij,ij->i", normal, view) < 0 if cam.perspective else normal[:, 2] < 0
        assert np.array_equal(area < 0, facing)
