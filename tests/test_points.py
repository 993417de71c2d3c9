"""Point rasterizer: rasterize_points / rasterize_points_naive (point_render.cpp:82-155) and
the backward to the points (splat_position_backward, point_render.cpp:302-338).

CPU: the C restatement (oracle/raster_oracle.c) is bit-identical to the reference's own rasterize_points and
rasterize_points_naive on test_point_render.cpp:24-43's scenes. GPU: fp64 payload bit-identical to the oracle,
fp32 within tolerance, naive == tiled, gradients vs the reference's splat_position_backward.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2007_08501_b200 import scenes as S
from tests._common import rel_err


def point_scenes(n=15):
    """test_point_render.cpp:24-43: Rng(83), 1-3 clouds of <= 200 points, 32/64 px, K 1/8, radius 0.02-0.15,
    tile 16/8, perspective (focal 1.5) or orthographic camera."""
    rng = S.Rng(83)
    for trial in range(n):
        b = 1 + rng.uniform_int(3)
        clouds = S.random_clouds(rng, b, 200)
        H = 32 if rng.uniform_int(2) == 0 else 64
        K = 1 if rng.uniform_int(2) == 0 else 8
        radius = rng.uniform(0.02, 0.15)
        tile = 16 if rng.uniform_int(2) == 0 else 8
        persp = rng.uniform_int(2) == 0
        cam = S.Camera.look_from_distance(3.0, True, 1.5) if persp else S.Camera.look_from_distance(3.0, False)
        yield trial, clouds, cam, H, K, radius, tile


def _packed(clouds):
    pts = np.concatenate(clouds, 0)
    num = np.array([len(c) for c in clouds], np.int64)
    first = np.concatenate([[0], np.cumsum(num)[:-1]]).astype(np.int64)
    return pts, first, num


def test_point_oracle_matches_reference(reflib, oracle):
    for trial, clouds, cam, H, K, radius, tile in point_scenes():
        pts, first, num = _packed(clouds)
        ndc = S.points_ndc(pts, cam)
        ref_t = reflib.rasterize_points(pts, num, cam.packed(), H, H, K, radius, tile=tile)
        ref_n = reflib.rasterize_points(pts, num, cam.packed(), H, H, K, radius, tile=tile, naive=True)
        orc_t = oracle.rasterize_points(ndc, first, num, H, H, K, radius, tile=tile, znear=cam.znear,
                                        clip_nonpositive_z=int(cam.perspective))
        orc_n = oracle.rasterize_points(ndc, first, num, H, H, K, radius, tile=0, znear=cam.znear,
                                        clip_nonpositive_z=int(cam.perspective))
        for a, b, name in zip(orc_t + orc_n, ref_t + ref_n, ["idx", "zbuf", "dists2"] * 2):
            assert np.array_equal(a, b), f"trial {trial}: {name} differs from the reference"
        assert (ref_t[0] >= 0).any()


def _settings(H, K, radius, tile, cam):
    from paper_2007_08501_b200 import PointRasterSettings

    return PointRasterSettings(image_size=H, points_per_pixel=K, radius=radius, bin_size=tile, znear=cam.znear,
                               clip_nonpositive_z=cam.perspective)


@pytest.mark.gpu
def test_points_bit_exact_vs_oracle(oracle, cuda):
    from paper_2007_08501_b200 import rasterize_points

    for trial, clouds, cam, H, K, radius, tile in point_scenes():
        pts, first, num = _packed(clouds)
        ndc = S.points_ndc(pts, cam)
        want = oracle.rasterize_points(ndc, first, num, H, H, K, radius, tile=tile, znear=cam.znear,
                                       clip_nonpositive_z=int(cam.perspective))
        x = torch.as_tensor(ndc, device=cuda)
        for bs in (tile, 0, 32):
            got = rasterize_points(x, first, num, _settings(H, K, radius, bs, cam), out_dtype=torch.float64)
            for g, w, name in zip(got, want, ("idx", "zbuf", "dists2")):
                assert np.array_equal(g.cpu().numpy(), w), f"trial {trial} bin {bs}: {name} differs"
        got32 = rasterize_points(x, first, num, _settings(H, K, radius, tile, cam))
        assert np.array_equal(got32[0].cpu().numpy(), want[0])
        np.testing.assert_allclose(got32[1].cpu().numpy().astype(np.float64), want[1], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(got32[2].cpu().numpy().astype(np.float64), want[2], rtol=1e-5, atol=1e-6)


@pytest.mark.gpu
def test_points_large_k_and_dense_cloud(oracle, cuda):
    """K beyond the register lists (generic local-memory path) and a dense cloud with many z ties."""
    from paper_2007_08501_b200 import rasterize_points

    rng = np.random.default_rng(4)
    pts = rng.standard_normal((6000, 3)) * 0.6
    pts[::3, 2] = pts[1::3, 2][: len(pts[::3])]  # exact z ties across points
    cam = S.bench_camera()
    ndc = S.points_ndc(pts, cam)
    first, num = np.array([0, 2500]), np.array([2500, 3500])
    for K in (1, 16, 40):
        want = oracle.rasterize_points(ndc, first, num, 48, 48, K, 0.08, tile=16, znear=cam.znear)
        got = rasterize_points(torch.as_tensor(ndc, device=cuda), first, num, _settings(48, K, 0.08, 16, cam),
                               out_dtype=torch.float64)
        for g, w in zip(got, want):
            assert np.array_equal(g.cpu().numpy(), w), f"K={K}"


@pytest.mark.gpu
@pytest.mark.parametrize("K", [1, 4])
def test_points_early_exit_bucket_bound(oracle, cuda, K):
    """Bins of thousands of points whose depths all fall in a sliver (one depth bucket of the bins' 1024-bucket
    order): the point fine stage stops streaming a bin once a lower bound of every remaining key exceeds every
    pixel's K-th depth. In bucket order the next key itself is NOT such a bound (nearer points of the same bucket
    can follow it); the stage uses the lower edge of the bucket two below the next entry's, from the (lo, scale)
    bucket map the sort wrote for the bin. Exiting at the next key fails this scene."""
    from paper_2007_08501_b200 import rasterize_points

    rng = np.random.default_rng(11)
    n = 6000  # a layer covering the whole image (ndc x = 2x/3 at depth 3): every pixel fills its K slots early
    pts = np.stack([rng.uniform(-1.8, 1.8, n), rng.uniform(-1.8, 1.8, n), rng.uniform(0.0, 5e-3, n)], 1)
    # far outliers stretch every bin's key range, so the whole dense layer lands in one of 1024 depth buckets
    far = np.stack([rng.uniform(-1.5, 1.5, 64), rng.uniform(-1.5, 1.5, 64), np.full(64, 5.0)], 1)
    pts = np.concatenate([pts, far])
    n = len(pts)
    cam = S.bench_camera()
    ndc = S.points_ndc(pts, cam)
    first, num = np.array([0]), np.array([n])
    want = oracle.rasterize_points(ndc, first, num, 32, 32, K, 0.2, tile=16, znear=cam.znear)
    got = rasterize_points(torch.as_tensor(ndc, device=cuda), first, num, _settings(32, K, 0.2, 16, cam),
                           out_dtype=torch.float64)
    for g, w in zip(got, want):
        assert np.array_equal(g.cpu().numpy(), w)


@pytest.mark.gpu
def test_points_backward_vs_reference(reflib, oracle, cuda):
    """splat_opacity -> d_alpha -> splat_position_backward (world space) vs the GPU chain."""
    from paper_2007_08501_b200 import rasterize_points, rasterize_points_backward, splat_position_backward, \
        world_to_points_ndc

    rng = S.Rng(97)
    clouds = S.random_clouds(rng, 2, 400)
    pts, first, num = _packed(clouds)
    cam = S.Camera.look_from_distance(3.0, True, 1.5)
    H, K, radius = 48, 8, 0.1
    rs = _settings(H, K, radius, 16, cam)
    ndc_gpu = world_to_points_ndc(torch.as_tensor(pts, device=cuda), cam)
    assert np.array_equal(ndc_gpu.cpu().numpy(), S.points_ndc(pts, cam))  # bit-identical projection
    frags = reflib.rasterize_points(pts, num, cam.packed(), H, H, K, radius)
    d_alpha = np.random.default_rng(5).standard_normal(frags[0].shape)
    d_ref = reflib.splat_position_backward(pts, num, cam.packed(), H, H, K, radius, frags, d_alpha)
    idx, zb, d2 = rasterize_points(ndc_gpu, first, num, rs, out_dtype=torch.float64)
    assert np.array_equal(idx.cpu().numpy(), frags[0])
    d_got = splat_position_backward(torch.as_tensor(pts, device=cuda), cam, ndc_gpu, first, num, rs, idx,
                                    torch.as_tensor(d_alpha, device=cuda)).cpu().numpy()
    assert np.abs(d_ref).max() > 0 and rel_err(d_got, d_ref) < 1e-10
    # zbuf cotangent path vs the oracle (fp32 cotangents)
    gz = np.random.default_rng(6).standard_normal(frags[0].shape).astype(np.float32)
    gd = np.random.default_rng(7).standard_normal(frags[0].shape).astype(np.float32)
    g = rasterize_points_backward(ndc_gpu, first, num, rs, idx, torch.as_tensor(gz, device=cuda),
                                  torch.as_tensor(gd, device=cuda)).cpu().numpy()
    g_w = oracle.rasterize_points_backward(S.points_ndc(pts, cam), frags[0], gz.astype(np.float64),
                                           gd.astype(np.float64))
    assert rel_err(g, g_w) < 1e-10


@pytest.mark.gpu
def test_points_errors(cuda):
    from paper_2007_08501_b200 import RangeError, ShapeError, rasterize_points

    x = torch.zeros((4, 3), dtype=torch.float64, device=cuda)
    cam = S.bench_camera()
    with pytest.raises(RangeError):
        rasterize_points(x, [0], [4], _settings(16, 200, 0.1, 16, cam))
    with pytest.raises(ShapeError):
        rasterize_points(x, [], [], _settings(16, 4, 0.1, 16, cam))
    with pytest.raises(ShapeError):
        rasterize_points(x[:, :2], [0], [4], _settings(16, 4, 0.1, 16, cam))
