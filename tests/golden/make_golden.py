"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libdr3d_ref.so, compiled from the
unmodified /root/reference sources by oracle/Makefile). Run in a container that has /root/reference:

    make -C oracle ref && python tests/golden/make_golden.py

Each fixture stores the boundary inputs (face_verts, mesh_to_face_first_idx, num_faces_per_mesh, settings)
and the reference's outputs, so parity can be checked on a box without the reference:
  kat.npz         point_triangle_dist2 / barycentric / clamp known answers (test_raster.cpp:11-111)
  c1.npz          C1: ico_sphere(3), 64x64, K=1, blur 0 (BASELINE configs[0])
  invariants.npz  ico_sphere(1), 48x48, K=8, blur 1e-3 (test_raster.cpp:151-192)
  soup_<t>.npz    acceptance scenes t (test_acceptance.cpp:143-183), one per camera/K/blur combination
  backward.npz    one-triangle scene, 12x12, K=2, blur 0.03, cotangents Rng(61) + reference d_verts
                  (test_raster.cpp:210-254)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefLib  # noqa: E402
from paper_2007_08501_b200 import scenes as S  # noqa: E402
from tests._common import acceptance_scenes  # noqa: E402


def save(name, meshes, cam, H, K, blur, tile, frags, extra=None):
    fv = S.face_verts(meshes, cam)
    d = dict(face_verts=fv, first=meshes.mesh_to_face_first_idx(), num=meshes.num_faces_per_mesh(),
             verts=meshes.verts_packed(), faces=meshes.faces_packed(), camera=cam.packed(),
             settings=np.array([H, H, K, tile], np.int64), blur=np.float64(blur),
             znear=np.float64(cam.znear), perspective=np.int64(cam.perspective),
             p2f=frags[0], zbuf=frags[1], bary=frags[2], dists=frags[3])
    d.update(extra or {})
    np.savez_compressed(os.path.join(HERE, name), **d)


def main():
    ref = RefLib()
    # KATs (test_raster.cpp:11-31, 99-111) evaluated by the reference library
    a, b, c = [0, 0], [1, 0], [0, 1]
    pts = [[0.25, 0.25], [-0.5, 0.5], [2, 0], [0.5, 0], [0.75, 0.75]]
    dist = [ref.point_triangle_dist2(p, a, b, c) for p in pts]
    deg = [ref.point_triangle_dist2(p, [0, 0], [1, 0], [2, 0]) for p in ([1, 0.5], [1, 0], [3, 0])]
    np.savez_compressed(os.path.join(HERE, "kat.npz"), tri=np.array([a, b, c], float), pts=np.array(pts, float),
                        dist=np.array(dist), deg_pts=np.array([[1, 0.5], [1, 0], [3, 0]], float),
                        deg_dist=np.array(deg))

    cam = S.bench_camera()
    m = S.ico_sphere(3)
    save("c1.npz", m, cam, 64, 1, 0.0, 16, ref.rasterize(ref.batch(m), cam.packed(), 64, 64, 1, 0.0, 16))

    cam2 = S.Camera.look_from_distance(3.0, True, 2.0)
    m = S.ico_sphere(1)
    save("invariants.npz", m, cam2, 48, 8, 1e-3, 16, ref.rasterize(ref.batch(m), cam2.packed(), 48, 48, 8, 1e-3, 16))

    keep = {1, 3, 4, 6, 9, 12, 15, 16, 18, 24, 27, 31}  # every (K, blur, camera) combination at 32/64 px
    for trial, m, cam3, H, K, blur, tile in acceptance_scenes(100):
        if trial in keep:
            save(f"soup_{trial:03d}.npz", m, cam3, H, K, blur, tile,
                 ref.rasterize(ref.batch(m), cam3.packed(), H, H, K, blur, tile))

    m = S.Meshes([np.array([[-0.8, -0.6, 0.1], [0.9, -0.5, 0.3], [0.0, 0.8, -0.2]])], [np.array([[0, 1, 2]])])
    cam4 = S.Camera.look_from_distance(3.0, True, 1.3)
    rb = ref.batch(m)
    fr = ref.rasterize(rb, cam4.packed(), 12, 12, 2, 0.03, 16)
    rng = S.Rng(61)
    n = fr[0].size
    wz = np.array([rng.normal() for _ in range(n)])
    wb = np.array([rng.normal() for _ in range(3 * n)])
    wd = np.array([rng.normal() for _ in range(n)])
    d_verts = ref.rasterize_backward(rb, cam4.packed(), 12, 12, 2, 0.03, fr, wz, wb, wd)
    save("backward.npz", m, cam4, 12, 2, 0.03, 16, fr, dict(d_zbuf=wz, d_bary=wb, d_dists=wd, d_verts=d_verts))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
