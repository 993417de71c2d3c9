"""Fused softmax render: the reference's differentiable softmax render op (grad.cpp:177-209 =
rasterize_meshes -> interpolate_face_attributes(vertex colours) -> softmax_blend, and its vjp through
softmax_blend_backward -> interpolate_face_attributes_backward -> rasterize_backward), checked against the
reference library composing exactly those functions (oracle/ref_shim.cpp ref_softmax_render*)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2007_08501_b200 import scenes as S
from tests._common import boundary, grad_close, parity_report, raster_settings, rel_err

pytestmark = pytest.mark.gpu

CASES = [("ico2", 48, 4, 2e-4, 1e-4, 1e-4), ("C2", 96, 8, 1e-4, 1e-4, 1e-4), ("C2g", 64, 8, 1e-4, 3e-4, 1e-2),
         ("ico2k1", 40, 1, 0.0, 1e-4, 1e-4), ("C2k20", 48, 20, 5e-4, 2e-4, 1e-3),
         ("C2k64", 40, 64, 9.2e-4, 1e-4, 1e-4),  # K > 16: the slot-compacted backward (5-pixel chunks at K=64)
         ("C2big", 256, 8, 1e-4, 1e-4, 1e-4)]  # enough 32-pixel groups for > 1 group per warp of a backward CTA


def _scene(name):
    return S.ico_sphere(2) if name.startswith("ico") else S.config_meshes("C2")


@pytest.mark.parametrize("name,H,K,blur,sigma,gamma", CASES)
def test_softmax_render_vs_reference(name, H, K, blur, sigma, gamma, reflib, cuda):
    from paper_2007_08501_b200 import BlendParams, rasterize_softmax, rasterize_softmax_backward

    m, cam = _scene(name), S.bench_camera()
    V = len(m.verts_packed())
    vc = np.random.default_rng(3).uniform(0.0, 1.0, (V, 3))
    bg = (0.25, 0.5, 0.75)
    rb = reflib.batch(m)
    img_ref, p2f_ref = reflib.softmax_render(rb, cam.packed(), H, H, K, blur, vc, sigma, gamma, bg)
    fv, first, num = boundary(m, cam)
    rs = raster_settings(H, K, blur, cam)
    bp = BlendParams(sigma=sigma, gamma=gamma, background_color=bg, znear=cam.znear, zfar=cam.zfar)
    dev = lambda a: torch.as_tensor(a, device=cuda)  # noqa: E731
    faces = m.faces_packed()
    p2f, img = rasterize_softmax(dev(fv), dev(first), dev(num), rs, bp, dev(vc), dev(faces))
    assert np.array_equal(p2f.cpu().numpy(), p2f_ref)
    np.testing.assert_allclose(img.cpu().numpy().astype(np.float64), img_ref, rtol=1e-5, atol=1e-6)
    assert np.any(np.all(img_ref == np.array(bg), -1))  # background pixels exist
    d_img = np.random.default_rng(5).standard_normal(img_ref.shape).astype(np.float32)
    dv_ref, dc_ref = reflib.softmax_render_backward(rb, cam.packed(), H, H, K, blur, vc, sigma, gamma,
                                                    d_img.astype(np.float64), bg)
    assert np.abs(dv_ref).max() > 0 and np.abs(dc_ref).max() > 0
    g_fv, g_vc = rasterize_softmax_backward(dev(fv), dev(first), dev(num), rs, bp, dev(vc), dev(faces), p2f,
                                            dev(d_img))
    d_got = S.scatter_face_grads(m, cam, g_fv.cpu().numpy())
    ev, ec = rel_err(d_got, dv_ref), rel_err(g_vc.cpu().numpy(), dc_ref)
    assert ev < 1e-4, f"{name}: d_verts rel err {ev:.2e}"
    ratio = grad_close(d_got, dv_ref, name)
    assert ec < 1e-6, f"{name}: d_colors rel err {ec:.2e}"
    parity_report(test="softmax", case=name, d_verts_rel_err=ev, d_verts_worst_err_over_bound=ratio,
                  d_colors_rel_err=ec)


def test_softmax_autograd_and_errors(cuda):
    from paper_2007_08501_b200 import BlendParams, RangeError, RasterizeSoftmax, rasterize_softmax

    m, cam = S.ico_sphere(2), S.bench_camera()
    fv, first, num = boundary(m, cam)
    rs = raster_settings(32, 4, 1e-4, cam)
    bp = BlendParams(znear=cam.znear, zfar=cam.zfar)
    V = len(m.verts_packed())
    x = torch.as_tensor(fv, device=cuda).requires_grad_(True)
    c = torch.rand((V, 3), dtype=torch.float64, device=cuda).requires_grad_(True)
    faces = torch.as_tensor(m.faces_packed(), device=cuda)
    img = RasterizeSoftmax.apply(x, c, faces, torch.as_tensor(first, device=cuda), torch.as_tensor(num, device=cuda),
                                 rs, bp)
    (img * img).sum().backward()
    assert torch.isfinite(x.grad).all() and x.grad.abs().sum() > 0 and c.grad.abs().sum() > 0
    with pytest.raises(RangeError):
        rasterize_softmax(torch.as_tensor(fv, device=cuda), first, num, rs, BlendParams(gamma=0.0), c, faces)
