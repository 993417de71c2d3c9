"""Fused silhouette consumer: silhouette_blend(rasterize_meshes(...)) forward and
rasterize_backward(0, 0, silhouette_blend_backward(...)) backward (shading.cpp:75-121, pipeline.cpp:153-162).

CPU: the C restatement (oracle/raster_oracle.c) vs the reference's own silhouette_blend / _backward.
GPU: the fused kernels vs the oracle chain, and end to end vs the reference library's world-space gradients.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2007_08501_b200 import scenes as S
from tests._common import boundary, grad_close, orc_settings, raster_settings, rel_err

SIGMA = 1e-4
GRAD_RTOL = 1e-4


def _ref_fragments(reflib, m, cam, H, K, blur):
    rb = reflib.batch(m)
    return rb, reflib.rasterize(rb, cam.packed(), H, H, K, blur)


@pytest.mark.parametrize("K,blur", [(8, 1e-4), (1, 0.0), (50, 9.2102e-4)])
def test_oracle_silhouette_matches_reference(reflib, oracle, K, blur):
    m, cam = S.synthetic_batch(3000.0, 1000.0, 3, 7), S.bench_camera()
    _, frags = _ref_fragments(reflib, m, cam, 48, K, blur)
    p2f, _, _, dists = frags
    a_ref = reflib.silhouette_blend(p2f, dists, SIGMA)
    a_orc = oracle.silhouette_blend(p2f, dists, SIGMA)
    assert np.array_equal(a_orc, a_ref)
    assert a_ref.max() > 0.5 and a_ref.min() == 0.0
    da = np.random.default_rng(3).standard_normal(a_ref.shape)
    da[0, :4] = 0.0  # d_alpha == 0 pixels are skipped (shading.cpp:102)
    dd_ref = reflib.silhouette_blend_backward(p2f, dists, SIGMA, da)
    dd_orc = oracle.silhouette_blend_backward(p2f, dists, SIGMA, da)
    assert np.array_equal(dd_orc, dd_ref)


def _gpu_sil(fv, first, num, rs, dev, sigma=SIGMA):
    from paper_2007_08501_b200 import rasterize_silhouette

    p2f, alpha = rasterize_silhouette(torch.as_tensor(fv, device=dev), torch.as_tensor(first, device=dev),
                                      torch.as_tensor(num, device=dev), rs, sigma)
    return p2f, alpha


CASES = [("C2", 128, 8, 1e-4, False), ("fit", 64, 4, 2e-4, False), ("k50", 64, 50, 9.2102e-4, False),
         ("C4flags", 96, 8, 1e-4, True)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,H,K,blur,flags", CASES)
def test_fused_silhouette_forward_and_backward(name, H, K, blur, flags, oracle, cuda):
    from paper_2007_08501_b200 import rasterize_silhouette_backward

    if name == "C2":
        m = S.config_meshes("C2")
    elif name == "fit":
        m = S.ico_sphere(2)
    else:
        m = S.rotated_cubes(4, 3, draw_faces=(1000.0, 20000.0))
    cam = S.bench_camera()
    fv, first, num = boundary(m, cam)
    kw = dict(persp_correct=1, cull=1) if flags else {}
    o = orc_settings(H, K, blur, cam, **kw)
    rs = raster_settings(H, K, blur, cam, persp_correct=flags, cull=flags)
    w_p2f, _, w_bary, w_d = oracle.forward(fv, first, num, o)
    p2f, alpha = _gpu_sil(fv, first, num, rs, cuda)
    assert np.array_equal(p2f.cpu().numpy(), w_p2f), f"{name}: pix_to_face differs from the oracle"
    w_alpha = oracle.silhouette_blend(w_p2f, w_d, SIGMA)
    np.testing.assert_allclose(alpha.cpu().numpy().astype(np.float64), w_alpha, rtol=1e-5, atol=1e-6)
    # backward: the reference fit loop's chain on the oracle
    da = np.random.default_rng(11).standard_normal(w_alpha.shape).astype(np.float32)
    da[..., ::7] = 0.0
    dd = oracle.silhouette_blend_backward(w_p2f, w_d, SIGMA, da.astype(np.float64))
    zeros = np.zeros_like(w_d)
    g_want = oracle.backward(fv, first, num, o, w_p2f, w_bary, zeros, np.zeros_like(w_bary), dd)
    g = rasterize_silhouette_backward(torch.as_tensor(fv, device=cuda), torch.as_tensor(first, device=cuda),
                                      torch.as_tensor(num, device=cuda), rs, SIGMA, p2f,
                                      torch.as_tensor(da, device=cuda)).cpu().numpy()
    assert np.abs(g_want).max() > 0
    assert rel_err(g, g_want) < GRAD_RTOL, f"{name}: grad rel err {rel_err(g, g_want):.2e}"
    # per element: the fp32-cotangent path evaluates the opacity sigmoid with fp32 exp (raster_bwd.cu), ~1e-7
    # relative per slot contribution, so the absolute term is 1e-6 of the largest gradient here (1e-8 for K3)
    grad_close(g, g_want, name, atol_scale=1e-6)
    assert np.all(g[..., 2] == 0.0)  # d_zbuf = d_bary = 0: no depth gradient


@pytest.mark.gpu
def test_fused_silhouette_end_to_end_vs_reference(reflib, cuda):
    """Reference: silhouette_blend(rasterize_meshes) -> silhouette_blend_backward -> rasterize_backward with
    zero d_zbuf/d_bary (pipeline.cpp:153-162) in world space vs the fused GPU path + vertex scatter."""
    from paper_2007_08501_b200 import rasterize_silhouette_backward

    m, cam = S.config_meshes("C2"), S.bench_camera()
    H, K, blur = 128, 8, 1e-4
    rb, frags = _ref_fragments(reflib, m, cam, H, K, blur)
    a_ref = reflib.silhouette_blend(frags[0], frags[3], SIGMA)
    da = (a_ref - 0.5).astype(np.float32)  # an IoU-like cotangent, dense on the rim band
    dd = reflib.silhouette_blend_backward(frags[0], frags[3], SIGMA, da.astype(np.float64))
    d_ref = reflib.rasterize_backward(rb, cam.packed(), H, H, K, blur, frags, np.zeros_like(frags[1]),
                                      np.zeros_like(frags[2]), dd)
    fv, first, num = boundary(m, cam)
    rs = raster_settings(H, K, blur, cam)
    p2f, alpha = _gpu_sil(fv, first, num, rs, cuda)
    assert np.array_equal(p2f.cpu().numpy(), frags[0])
    np.testing.assert_allclose(alpha.cpu().numpy().astype(np.float64), a_ref, rtol=1e-5, atol=1e-6)
    g = rasterize_silhouette_backward(torch.as_tensor(fv, device=cuda), torch.as_tensor(first, device=cuda),
                                      torch.as_tensor(num, device=cuda), rs, SIGMA, p2f,
                                      torch.as_tensor(da, device=cuda)).cpu().numpy()
    d_got = S.scatter_face_grads(m, cam, g)
    assert rel_err(d_got, d_ref) < GRAD_RTOL


@pytest.mark.gpu
def test_fused_silhouette_autograd_and_errors(cuda):
    from paper_2007_08501_b200 import RangeError, RasterizeSilhouette, rasterize_silhouette

    m, cam = S.ico_sphere(2), S.bench_camera()
    fv, first, num = boundary(m, cam)
    rs = raster_settings(32, 4, 1e-4, cam)
    x = torch.as_tensor(fv, device=cuda).requires_grad_(True)
    alpha = RasterizeSilhouette.apply(x, torch.as_tensor(first, device=cuda), torch.as_tensor(num, device=cuda), rs,
                                      SIGMA)
    (alpha * alpha).sum().backward()
    assert x.grad is not None and torch.isfinite(x.grad).all() and x.grad.abs().sum() > 0
    with pytest.raises(RangeError):
        rasterize_silhouette(torch.as_tensor(fv, device=cuda), first, num, rs, sigma=0.0)
    # no pix_to_face requested: alpha alone is identical
    _, a1 = rasterize_silhouette(torch.as_tensor(fv, device=cuda), first, num, rs, SIGMA, want_pix_to_face=False)
    _, a2 = rasterize_silhouette(torch.as_tensor(fv, device=cuda), first, num, rs, SIGMA)
    assert torch.equal(a1, a2)


@pytest.mark.gpu
@pytest.mark.parametrize("K,blur,sigma", [(8, 1e-4, SIGMA), (24, 4e-3, 2e-3)])
def test_fused_silhouette_f64_vs_reference(reflib, cuda, K, blur, sigma):
    """fp64 entry points (the fit loop's): alpha to a few ulps of silhouette_blend over the reference's fp64
    MeshFragments, world-space gradients to 1e-10 of the reference chain."""
    from paper_2007_08501_b200 import rasterize_silhouette, rasterize_silhouette_backward

    m, cam = S.config_meshes("C2"), S.bench_camera()
    H = 96
    rb, frags = _ref_fragments(reflib, m, cam, H, K, blur)
    a_ref = reflib.silhouette_blend(frags[0], frags[3], sigma)
    da = a_ref - 0.5
    dd = reflib.silhouette_blend_backward(frags[0], frags[3], sigma, da)
    d_ref = reflib.rasterize_backward(rb, cam.packed(), H, H, K, blur, frags, np.zeros_like(frags[1]),
                                      np.zeros_like(frags[2]), dd)
    fv, first, num = boundary(m, cam)
    rs = raster_settings(H, K, blur, cam)
    fvt, ft, nt = (torch.as_tensor(x, device=cuda) for x in (fv, first, num))
    p2f, alpha = rasterize_silhouette(fvt, ft, nt, rs, sigma, out_dtype=torch.float64)
    assert alpha.dtype == torch.float64
    assert np.array_equal(p2f.cpu().numpy(), frags[0])
    np.testing.assert_allclose(alpha.cpu().numpy(), a_ref, rtol=1e-13, atol=1e-15)
    g = rasterize_silhouette_backward(fvt, ft, nt, rs, sigma, p2f, torch.as_tensor(da, device=cuda)).cpu().numpy()
    assert rel_err(S.scatter_face_grads(m, cam, g), d_ref) < 1e-10
