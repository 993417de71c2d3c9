"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle (oracle/raster_oracle.c, itself pinned
bit-identical to the reference by tests/test_oracle_pin.py).

Bar (BASELINE.json north_star): pix_to_face bit-exact; zbuf / bary / dists within 1e-5 rel / 1e-6 abs for the
fp32 payload (the fp64 payload variant is checked BIT-EXACT); face_verts gradients within 1e-4 relative.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from paper_2007_08501_b200 import scenes as S
from tests._common import (acceptance_scenes, boundary, cotangents, fast_cotangents, grad_close, orc_settings,
                           raster_settings, raster_test_scenes, rel_err)

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6  # fragment payload tolerance (fp32 outputs vs fp64 oracle)
GRAD_RTOL = 1e-4


def gpu_fwd(fv, first, num, rs, dev, out_dtype=torch.float32):
    from paper_2007_08501_b200 import rasterize_meshes

    out = rasterize_meshes(torch.as_tensor(fv, device=dev), torch.as_tensor(first, device=dev),
                           torch.as_tensor(num, device=dev), rs, out_dtype=out_dtype)
    return [t.cpu().numpy() for t in out]


def gpu_bwd(fv, first, num, rs, dev, p2f, bary, dz, db, dd, dtype=torch.float32):
    from paper_2007_08501_b200 import rasterize_meshes_backward

    shp = p2f.shape
    t = lambda a, s: torch.as_tensor(np.asarray(a).reshape(s), dtype=dtype, device=dev)  # noqa: E731
    g = rasterize_meshes_backward(torch.as_tensor(fv, device=dev), torch.as_tensor(first, device=dev),
                                  torch.as_tensor(num, device=dev), rs, torch.as_tensor(p2f, device=dev),
                                  t(bary, shp + (3,)), t(dz, shp), t(db, shp + (3,)), t(dd, shp))
    return g.cpu().numpy()


def assert_frag_exact(got, want, msg=""):
    for name, g, w in zip(("pix_to_face", "zbuf", "bary", "dists"), got, want):
        assert np.array_equal(g, w), f"{msg}: {name} differs at {np.argwhere(g != w)[:5].tolist()}"


def assert_frag_close(got, want, msg=""):
    p2f_g, z_g, b_g, d_g = got
    p2f_w, z_w, b_w, d_w = want
    assert np.array_equal(p2f_g, p2f_w), f"{msg}: pix_to_face differs at {np.argwhere(p2f_g != p2f_w)[:5].tolist()}"
    for name, g, w in (("zbuf", z_g, z_w), ("bary", b_g, b_w), ("dists", d_g, d_w)):
        np.testing.assert_allclose(g.astype(np.float64), w, rtol=RTOL, atol=ATOL, err_msg=f"{msg}: {name}")


# -------------------------------------------------------------------------------------------------
# reference scenes: fp64 payload bit-exact, fp32 within tolerance, naive == binned


@pytest.mark.parametrize("which", ["raster", "acceptance"])
def test_reference_scenes_bit_exact(which, oracle, cuda):
    gen = raster_test_scenes(20) if which == "raster" else acceptance_scenes(100)
    for trial, m, cam, H, K, blur, tile in gen:
        fv, first, num = boundary(m, cam)
        want = oracle.forward(fv, first, num, orc_settings(H, K, blur, cam))
        for bs in (tile, 0):
            rs = raster_settings(H, K, blur, cam, bin_size=bs)
            got64 = gpu_fwd(fv, first, num, rs, cuda, torch.float64)
            assert_frag_exact(got64, want, f"{which} trial {trial} bin {bs}")
        got32 = gpu_fwd(fv, first, num, raster_settings(H, K, blur, cam, bin_size=tile), cuda)
        assert_frag_close(got32, want, f"{which} trial {trial} fp32")


def test_c1_ico_sphere(oracle, cuda):
    m, cam = S.ico_sphere(3), S.bench_camera()
    fv, first, num = boundary(m, cam)
    want = oracle.forward(fv, first, num, orc_settings(64, 1, 0.0, cam))
    for bs in (16, 8, 0, 64, 5):
        got = gpu_fwd(fv, first, num, raster_settings(64, 1, 0.0, cam, bin_size=bs), cuda, torch.float64)
        assert_frag_exact(got, want, f"C1 bin {bs}")
    assert (want[0] >= 0).sum() == 1600  # 1,600 occupied slots of 4,096


def test_slot_invariants_and_blur(oracle, cuda):
    """test_raster.cpp:151-208 on the GPU path."""
    m, cam = S.ico_sphere(1), S.Camera.look_from_distance(3.0, True, 2.0)
    fv, first, num = boundary(m, cam)
    p2f, z, b, d = gpu_fwd(fv, first, num, raster_settings(48, 8, 1e-3, cam), cuda, torch.float64)
    occ = p2f >= 0
    assert occ.any()
    # occupied slots form a prefix
    assert not np.any(~occ[..., :-1] & occ[..., 1:])
    assert np.all(d[occ] <= 1e-3) and np.all(z[occ] >= cam.znear)
    assert np.all(b[occ] >= 0) and np.allclose(b[occ].sum(-1), 1.0, atol=1e-9)
    both = occ[..., 1:] & occ[..., :-1]
    zp, zc, ip, ic = z[..., :-1], z[..., 1:], p2f[..., :-1], p2f[..., 1:]
    assert np.all(((zp < zc) | ((zp == zc) & (ip < ic)))[both])
    tight = gpu_fwd(fv, first, num, raster_settings(64, 1, 0.0, cam), cuda)[0]
    loose = gpu_fwd(fv, first, num, raster_settings(64, 1, 5e-3, cam), cuda)[0]
    assert (loose >= 0).sum() > (tight >= 0).sum()


def test_overflow_spill_does_not_change_results(oracle, cuda):
    """max_faces_per_bin below the real bin sizes: the spill path must give identical fragments."""
    m = S.synthetic_batch(11000.0, 18000.0 / (2.0 * math.sqrt(3.0)), 3, 0)
    cam = S.bench_camera()
    fv, first, num = boundary(m, cam)
    want = gpu_fwd(fv, first, num, raster_settings(96, 4, 1e-4, cam, bin_size=0), cuda, torch.float64)
    for cap in (1, 7, 64, 100000):
        got = gpu_fwd(fv, first, num, raster_settings(96, 4, 1e-4, cam, bin_size=16, cap=cap), cuda, torch.float64)
        assert_frag_exact(got, want, f"cap {cap}")


def test_edge_cases(oracle, cuda):
    from paper_2007_08501_b200 import MeshIndexError, RangeError, ShapeError, rasterize_meshes

    cam = S.bench_camera()
    # zero-face mesh in the middle of the batch, K larger than the coverage, non-square image
    m = S.Meshes()
    m.extend(S.ico_sphere(1))
    m.verts.append(np.zeros((3, 3)))
    m.faces.append(np.zeros((0, 3), dtype=np.int64))
    m.extend(S.cube(0.7, 2))
    fv, first, num = boundary(m, cam)
    for H, W in ((40, 24), (17, 33)):
        want = oracle.forward(fv, first, num, orc_settings(H, 37, 2e-3, cam, W=W))
        got = gpu_fwd(fv, first, num, raster_settings(H, 37, 2e-3, cam, W=W, bin_size=8), cuda, torch.float64)
        assert_frag_exact(got, want, f"edge {H}x{W}")
        assert np.all(got[0][1] == -1) and np.all(got[1][1] == -1.0)
    # negative blur keeps the reference quirk (inflate clamps to 0, compare stays raw, MR:103,171)
    want = oracle.forward(fv, first, num, orc_settings(32, 2, -1e-4, cam))
    got = gpu_fwd(fv, first, num, raster_settings(32, 2, -1e-4, cam), cuda, torch.float64)
    assert_frag_exact(got, want, "negative blur")
    # non-contiguous / overlapping mesh ranges are taken literally
    first2, num2 = np.array([5, 0, 3]), np.array([10, 4, 2])
    want = oracle.forward(fv, first2, num2, orc_settings(32, 3, 1e-3, cam))
    got = gpu_fwd(fv, first2, num2, raster_settings(32, 3, 1e-3, cam), cuda, torch.float64)
    assert_frag_exact(got, want, "ranges")
    fvt = torch.as_tensor(fv, device=cuda)
    with pytest.raises(ShapeError):
        rasterize_meshes(fvt, torch.zeros(0, dtype=torch.int64), torch.zeros(0, dtype=torch.int64))
    with pytest.raises(MeshIndexError):
        rasterize_meshes(fvt, [0], [len(fv) + 1])
    with pytest.raises(RangeError):
        rasterize_meshes(fvt, [0], [3], faces_per_pixel=0)


def test_non_finite_and_degenerate_faces_are_culled(oracle, cuda):
    cam = S.bench_camera()
    m = S.ico_sphere(1)
    fv, first, num = boundary(m, cam)
    fv = fv.copy()
    fv[3, 1, 0] = np.nan
    fv[7, 2, 1] = np.inf
    fv[9] = fv[9, 0]  # all three vertices equal -> zero area (MR:114)
    want = oracle.forward(fv, first, num, orc_settings(48, 4, 1e-3, cam))
    got = gpu_fwd(fv, first, num, raster_settings(48, 4, 1e-3, cam), cuda, torch.float64)
    assert_frag_exact(got, want, "non-finite")
    assert not np.isin([3, 7, 9], got[0]).any()


@pytest.mark.parametrize("persp,clip,cull", [(1, 1, 0), (0, 0, 0), (1, 0, 1), (0, 1, 1)])
def test_builder_defined_flags(persp, clip, cull, oracle, cuda):
    """perspective_correct / clip_barycentric_coords=0 / cull_backfaces: pinned by the oracle restatement."""
    m = S.rotated_cubes(4, 2, draw_faces=(200.0, 3000.0))
    cam = S.bench_camera()
    fv, first, num = boundary(m, cam)
    o = orc_settings(64, 8, 1e-3, cam, persp_correct=persp, clip=clip, cull=cull)
    want = oracle.forward(fv, first, num, o)
    rs = raster_settings(64, 8, 1e-3, cam, persp_correct=bool(persp), clip=bool(clip), cull=bool(cull))
    got = gpu_fwd(fv, first, num, rs, cuda, torch.float64)
    assert_frag_exact(got, want, f"flags {persp}{clip}{cull}")
    dz, db, dd = fast_cotangents(want[0].size, 3)
    g_want = oracle.backward(fv, first, num, o, want[0], want[2], dz, db, dd)
    g_got = gpu_bwd(fv, first, num, rs, cuda, got[0], got[2], dz, db, dd, torch.float64)
    assert rel_err(g_got, g_want) < 1e-9
    grad_close(g_got, g_want, f"flags {persp}{clip}{cull}")


def test_forward_rerun_identical(cuda):
    m, cam = S.config_meshes("C2"), S.bench_camera()
    fv, first, num = boundary(m, cam)
    rs = raster_settings(128, 8, 1e-4, cam)
    a = gpu_fwd(fv, first, num, rs, cuda)
    b = gpu_fwd(fv, first, num, rs, cuda)
    assert_frag_exact(a, b, "rerun")


# -------------------------------------------------------------------------------------------------
# backward


def test_c2_forward_backward(oracle, cuda):
    """C2: 8 heterogeneous meshes, 128^2, K=8, blur 1e-4, reference cotangent stream Rng(1)."""
    m, cam = S.config_meshes("C2"), S.bench_camera()
    fv, first, num = boundary(m, cam)
    o = orc_settings(128, 8, 1e-4, cam)
    want = oracle.forward(fv, first, num, o)
    got = gpu_fwd(fv, first, num, raster_settings(128, 8, 1e-4, cam), cuda)
    assert_frag_close(got, want, "C2")
    assert (want[0] >= 0).sum() == 570472
    dz, db, dd = cotangents(want[0].size)
    dz32, db32, dd32 = (x.astype(np.float32) for x in (dz, db, dd))
    g_want = oracle.backward(fv, first, num, o, want[0], want[2], dz32.astype(np.float64), db32.astype(np.float64),
                             dd32.astype(np.float64))
    g_got = gpu_bwd(fv, first, num, raster_settings(128, 8, 1e-4, cam), cuda, got[0], got[2], dz32, db32, dd32)
    assert rel_err(g_got, g_want) < GRAD_RTOL
    grad_close(g_got, g_want, "C2 fp32")
    # fp64 variant: same inputs as the oracle, agreement to accumulation order
    g64 = gpu_bwd(fv, first, num, raster_settings(128, 8, 1e-4, cam), cuda, want[0], want[2], dz, db, dd,
                  torch.float64)
    g_w64 = oracle.backward(fv, first, num, o, want[0], want[2], dz, db, dd)
    assert rel_err(g64, g_w64) < 1e-12
    grad_close(g64, g_w64, "C2 fp64")


def test_backward_end_to_end_vs_reference(reflib, oracle, cuda):
    """GPU grads -> vertex scatter -> world_to_ndc_backward == reference rasterize_backward (MR:329-403)."""
    m, cam = S.config_meshes("C2"), S.bench_camera()
    fv, first, num = boundary(m, cam)
    rb = reflib.batch(m)
    frags = reflib.rasterize(rb, cam.packed(), 128, 128, 8, 1e-4)
    dz, db, dd = cotangents(frags[0].size)
    d_ref = reflib.rasterize_backward(rb, cam.packed(), 128, 128, 8, 1e-4, frags, dz, db, dd)
    g = gpu_bwd(fv, first, num, raster_settings(128, 8, 1e-4, cam), cuda, frags[0], frags[2], dz, db, dd,
                torch.float64)
    d_got = S.scatter_face_grads(m, cam, g)
    assert rel_err(d_got, d_ref) < 1e-10
    grad_close(d_got, d_ref, "C2 world d_verts vs reference")


def test_backward_finite_differences(cuda):
    """test_raster.cpp:210-254 through the GPU path: one triangle, 12^2, K=2, blur 0.03, eps 1e-6."""
    m = S.Meshes([np.array([[-0.8, -0.6, 0.1], [0.9, -0.5, 0.3], [0.0, 0.8, -0.2]])], [np.array([[0, 1, 2]])])
    cam = S.Camera.look_from_distance(3.0, True, 1.3)
    rs = raster_settings(12, 2, 0.03, cam)
    fv, first, num = boundary(m, cam)
    base = gpu_fwd(fv, first, num, rs, cuda, torch.float64)
    rng = S.Rng(61)
    n = base[0].size
    wz = np.array([rng.normal() for _ in range(n)])
    wb = np.array([rng.normal() for _ in range(3 * n)])
    wd = np.array([rng.normal() for _ in range(n)])

    def scalar(verts):
        mm = S.Meshes([verts], m.faces)
        p2f, z, b, d = gpu_fwd(*boundary(mm, cam), rs, cuda, torch.float64)
        occ = (p2f >= 0).reshape(-1)
        return float((wz * z.reshape(-1) + wd * d.reshape(-1))[occ].sum()
                     + (wb.reshape(-1, 3) * b.reshape(-1, 3))[occ].sum())

    g = gpu_bwd(fv, first, num, rs, cuda, base[0], base[2], wz, wb, wd, torch.float64)
    d_verts = S.scatter_face_grads(m, cam, g)
    v0 = m.verts[0]
    eps = 1e-6
    for i in range(3):
        for ax in range(3):
            vp, vm = v0.copy(), v0.copy()
            vp[i, ax] += eps
            vm[i, ax] -= eps
            fd = (scalar(vp) - scalar(vm)) / (2 * eps)
            an = d_verts[i, ax]
            assert abs(fd - an) / max(abs(fd), abs(an), 1e-6) <= 2e-3


def test_autograd_function(cuda):
    from paper_2007_08501_b200 import RasterizeMeshes

    m, cam = S.ico_sphere(2), S.bench_camera()
    fv, first, num = boundary(m, cam)
    rs = raster_settings(32, 4, 1e-3, cam)
    x = torch.as_tensor(fv, device=cuda).requires_grad_(True)
    p2f, z, b, d = RasterizeMeshes.apply(x, torch.as_tensor(first, device=cuda), torch.as_tensor(num, device=cuda), rs)
    loss = (z * (p2f >= 0)).sum() + d.sum() + b[..., 0].sum()
    loss.backward()
    assert x.grad is not None and torch.isfinite(x.grad).all() and x.grad.abs().sum() > 0


# -------------------------------------------------------------------------------------------------
# BASELINE configs at full size


def _mesh_subset(first, num, idx):
    return first[idx], num[idx]


@pytest.mark.slow
def test_c3_large_sphere_with_overflow(oracle, cuda):
    """C3: 1.31M faces, 512^2, K=1, bin 32; max_faces_per_bin below the largest bin forces the spill path."""
    from paper_2007_08501_b200 import bin_stats, rasterize_meshes, workspace_bytes

    m, cam = S.config_meshes("C3"), S.bench_camera()
    fv, first, num = boundary(m, cam)
    want = oracle.forward(fv, first, num, orc_settings(512, 1, 0.0, cam))
    assert (want[0] >= 0).sum() == 102960
    for cap in (2048, 10000, 0):
        rs = raster_settings(512, 1, 0.0, cam, bin_size=32, cap=cap)
        ws = torch.empty(workspace_bytes(1, len(fv), rs), dtype=torch.uint8, device=cuda)
        out = rasterize_meshes(torch.as_tensor(fv, device=cuda), torch.as_tensor(first, device=cuda),
                               torch.as_tensor(num, device=cuda), rs, workspace=ws)
        st = bin_stats(1, len(fv), rs, ws)
        if cap == 2048:
            assert st["overflowed"] > 0
        assert_frag_close([t.cpu().numpy() for t in out], want, f"C3 cap {cap}")


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_full_config_properties_and_mesh_sample(cfg, oracle, cuda):
    """C4 / C5 at full size: size-independent slot invariants everywhere + oracle parity on a mesh sample."""
    c = S.CONFIGS[cfg]
    m, cam = S.config_meshes(cfg), S.bench_camera()
    fv, first, num = boundary(m, cam)
    H, K, blur = c["image"], c["K"], c["blur"]
    persp, cull = bool(c.get("perspective_correct", False)), bool(c.get("cull_backfaces", False))
    rs = raster_settings(H, K, blur, cam, persp_correct=persp, cull=cull)
    p2f, z, b, d = gpu_fwd(fv, first, num, rs, cuda)
    occ = p2f >= 0
    assert not np.any(~occ[..., :-1] & occ[..., 1:])
    assert np.all(d[occ] <= blur * (1 + 1e-6)) and np.all(z[occ] >= cam.znear * (1 - 1e-6))
    assert np.allclose(b[occ].sum(-1), 1.0, atol=1e-5)
    for bidx in (0, len(first) // 2, len(first) - 1):
        f_, n_ = first[[bidx]], num[[bidx]]
        o = orc_settings(H, K, blur, cam, persp_correct=int(persp), cull=int(cull))
        want = oracle.forward(fv, f_, n_, o)
        got = [a[bidx:bidx + 1] for a in (p2f, z, b, d)]
        assert_frag_close(got, want, f"{cfg} mesh {bidx}")
        if bidx == 0:
            S_ = want[0].size
            dz, db, dd = (x.astype(np.float32) for x in fast_cotangents(S_, 5))
            g_w = oracle.backward(fv, f_, n_, o, want[0], want[2], dz.astype(np.float64), db.astype(np.float64),
                                  dd.astype(np.float64))
            g_g = gpu_bwd(fv, f_, n_, rs, cuda, got[0], got[2], dz, db, dd)
            sl = slice(int(f_[0]), int(f_[0] + n_[0]))
            assert rel_err(g_g[sl], g_w[sl]) < GRAD_RTOL
            grad_close(g_g[sl], g_w[sl], f"{cfg} mesh 0")


# -------------------------------------------------------------------------------------------------
# camera side (world_to_ndc + gather, scatter + world_to_ndc_backward) on the GPU


def test_world_to_face_verts_bit_exact(cuda):
    from paper_2007_08501_b200 import MeshIndexError, world_to_face_verts

    m = S.config_meshes("C2")
    for cam in (S.bench_camera(), S.Camera.look_from_distance(3.0, False),
                S.Camera(rotation=S.axis_angle((0.3, -1.0, 0.2), 0.7), translation=(0.1, -0.2, 1.2),
                         focal_length=1.7, principal_point=(0.05, -0.02))):
        got = world_to_face_verts(torch.as_tensor(m.verts_packed(), device=cuda),
                                  torch.as_tensor(m.faces_packed(), device=cuda), cam).cpu().numpy()
        assert np.array_equal(got, S.face_verts(m, cam))
    with pytest.raises(MeshIndexError):
        bad = m.faces_packed().copy()
        bad[5, 1] = len(m.verts_packed())
        world_to_face_verts(torch.as_tensor(m.verts_packed(), device=cuda), torch.as_tensor(bad, device=cuda),
                            S.bench_camera())


def test_face_verts_backward_matches_host_chain(cuda):
    from paper_2007_08501_b200 import face_verts_backward

    m = S.config_meshes("C2")
    g = np.random.default_rng(7).standard_normal((len(m.faces_packed()), 3, 3))
    for cam in (S.bench_camera(), S.Camera.look_from_distance(3.0, False)):
        got = face_verts_backward(torch.as_tensor(m.verts_packed(), device=cuda),
                                  torch.as_tensor(m.faces_packed(), device=cuda), cam,
                                  torch.as_tensor(g, device=cuda)).cpu().numpy()
        want = S.scatter_face_grads(m, cam, g)
        assert rel_err(got, want) < 1e-12


def test_div_free_paths_and_rerun_backward_tolerance(cuda, oracle):
    """Backward on C1-like scene with fp64 inputs: GPU vs oracle to accumulation order only."""
    m, cam = S.ico_sphere(3), S.bench_camera()
    fv, first, num = boundary(m, cam)
    o = orc_settings(64, 4, 5e-3, cam)
    fr = oracle.forward(fv, first, num, o)
    dz, db, dd = fast_cotangents(fr[0].size, 11)
    want = oracle.backward(fv, first, num, o, fr[0], fr[2], dz, db, dd)
    got = gpu_bwd(fv, first, num, raster_settings(64, 4, 5e-3, cam), cuda, fr[0], fr[2], dz, db, dd, torch.float64)
    assert rel_err(got, want) < 1e-12


def test_host_pipeline_matches_device_calls(cuda):
    """HostPipeline (pinned host in/out, mesh groups streamed over 3 CUDA streams) == plain device calls."""
    from paper_2007_08501_b200 import rasterize_meshes, rasterize_meshes_backward
    from paper_2007_08501_b200.pipeline import HostPipeline

    m, cam = S.config_meshes("C2"), S.bench_camera()
    fv, first, num = boundary(m, cam)
    rs = raster_settings(128, 8, 1e-4, cam)
    N, F = len(num), len(fv)
    g = np.random.default_rng(3)
    cot = [torch.as_tensor(g.standard_normal(s), dtype=torch.float32) for s in
           ((N, 128, 128, 8), (N, 128, 128, 8, 3), (N, 128, 128, 8))]
    pipe = HostPipeline(first, num, rs, F, cuda, n_groups=3)
    from paper_2007_08501_b200.pipeline import contiguous_groups, transfer_costs

    assert pipe.groups == contiguous_groups(transfer_costs(num, 128 * 128 * 8, True), 3, 2)  # native == Python rule
    out_h = (torch.empty((N, 128, 128, 8), dtype=torch.int64).pin_memory(),
             torch.empty((N, 128, 128, 8), dtype=torch.float32).pin_memory(),
             torch.empty((N, 128, 128, 8, 3), dtype=torch.float32).pin_memory(),
             torch.empty((N, 128, 128, 8), dtype=torch.float32).pin_memory())
    grad_h = torch.empty((F, 3, 3), dtype=torch.float64).pin_memory()
    for _ in range(2):
        pipe.run(torch.as_tensor(fv).pin_memory(), out_h, tuple(c.pin_memory() for c in cot), grad_h)
        torch.cuda.synchronize()
    fvd = torch.as_tensor(fv, device=cuda)
    ref = rasterize_meshes(fvd, torch.as_tensor(first, device=cuda), torch.as_tensor(num, device=cuda), rs)
    for a, b in zip(out_h, ref):
        assert torch.equal(a, b.cpu())
    gref = rasterize_meshes_backward(fvd, torch.as_tensor(first, device=cuda), torch.as_tensor(num, device=cuda), rs,
                                     ref[0], ref[2], *(c.to(cuda) for c in cot))
    assert rel_err(grad_h.numpy(), gref.cpu().numpy()) < 1e-12


def test_backward_rejects_host_cotangents(cuda):
    """Cotangents in host memory (pageable: would fault; page-locked: read over PCIe, measured slower than copying)
    are rejected by the C-ABI (DR_ERR_USAGE)."""
    from paper_2007_08501_b200 import UsageError, rasterize_meshes, rasterize_meshes_backward

    m, cam = S.ico_sphere(1), S.bench_camera()
    fv, first, num = boundary(m, cam)
    rs = raster_settings(32, 2, 1e-4, cam)
    fvd, fd, nd = (torch.as_tensor(x, device=cuda) for x in (fv, first, num))
    p2f, zbuf, bary, dists = rasterize_meshes(fvd, fd, nd, rs)
    for pin in (False, True):
        mk = (lambda s: torch.zeros(s).pin_memory()) if pin else torch.zeros  # noqa: E731
        with pytest.raises(UsageError):
            rasterize_meshes_backward(fvd, fd, nd, rs, p2f, bary, mk(tuple(zbuf.shape)), mk(tuple(bary.shape)),
                                      mk(tuple(dists.shape)))


def test_grouped_exact_division_is_ieee(cuda):
    """xdiv_* (raster_math.cuh) == IEEE a/b bit for bit on hard cases: every selection-path quotient uses it."""
    import ctypes as C

    from paper_2007_08501_b200 import _lib

    L = _lib.load()
    bad = C.c_uint64(0)
    ab = (C.c_double * 2)()
    for seed in (1, 2, 3):
        assert L.dr_selftest_division(1 << 27, seed, C.byref(bad), ab) == 0
        assert bad.value == 0, f"grouped division differs from IEEE for a={ab[0]!r}, b={ab[1]!r}"
