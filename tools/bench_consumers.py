"""Fused vs unfused silhouette consumer on a bench config, one GPU.

  python tools/bench_consumers.py [--config C4] [--steps 10] [--warmup 3]

fused:    rasterize_silhouette + rasterize_silhouette_backward (alpha / pix_to_face only in HBM)
unfused:  rasterize_meshes -> silhouette_blend in torch ops (fp64) -> autograd d_dists ->
          rasterize_meshes_backward (fragments + cotangents round-trip through HBM)
fragments: the bench step (rasterize_meshes + rasterize_meshes_backward with random cotangents), for scale.
softmax:  the same comparison for the softmax render (vertex colours + softmax_blend, grad.cpp:177-209); the
          unfused arm's torch ops skip the reference's exact tie rule for zinv_max's argmax (timing arm only).
Prints one JSON line with ms per step of each and the kernels' share.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import config_settings  # noqa: E402
from paper_2007_08501_b200 import (rasterize_meshes, rasterize_meshes_backward, rasterize_silhouette,  # noqa: E402
                                   rasterize_silhouette_backward, scenes as S, workspace_bytes)


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sigma", type=float, default=1e-4)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    m, cam = S.config_meshes(a.config), S.bench_camera()
    rs = config_settings(a.config)
    fv = torch.as_tensor(S.face_verts(m, cam), device=dev)
    first = torch.as_tensor(m.mesh_to_face_first_idx(), device=dev)
    num = torch.as_tensor(m.num_faces_per_mesh(), device=dev)
    N, F = int(first.numel()), int(fv.shape[0])
    H, W = rs.hw
    K = rs.faces_per_pixel
    ws = torch.empty(workspace_bytes(N, F, rs), dtype=torch.uint8, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    d_alpha = torch.randn((N, H, W), generator=g, device=dev)
    dz = torch.randn((N, H, W, K), generator=g, device=dev)
    db = torch.randn((N, H, W, K, 3), generator=g, device=dev)
    dd = torch.randn((N, H, W, K), generator=g, device=dev)

    def fused():
        p2f, alpha = rasterize_silhouette(fv, first, num, rs, a.sigma, workspace=ws)
        return rasterize_silhouette_backward(fv, first, num, rs, a.sigma, p2f, d_alpha)

    def unfused():
        p2f, zbuf, bary, dists = rasterize_meshes(fv, first, num, rs, workspace=ws)
        d = dists.double().requires_grad_(True)
        occ = p2f >= 0
        prob = torch.sigmoid(-d / a.sigma)
        alpha = 1.0 - torch.where(occ, 1.0 - prob, torch.ones_like(prob)).prod(-1)
        (gd,) = torch.autograd.grad(alpha, d, d_alpha.double())
        gd = torch.where(occ, gd, torch.zeros_like(gd)).float()
        return rasterize_meshes_backward(fv, first, num, rs, p2f, bary, torch.zeros_like(zbuf),
                                         torch.zeros_like(bary), gd)

    def fragments():
        p2f, zbuf, bary, dists = rasterize_meshes(fv, first, num, rs, workspace=ws)
        return rasterize_meshes_backward(fv, first, num, rs, p2f, bary, dz, db, dd)

    # softmax render (grad.cpp:177-209): vertex colours interpolated with the clamped barycentrics, softmax blend
    from paper_2007_08501_b200 import BlendParams, rasterize_softmax, rasterize_softmax_backward

    V = len(m.verts_packed())
    vc = torch.rand((V, 3), generator=g, device=dev, dtype=torch.float64)
    faces = torch.as_tensor(m.faces_packed(), device=dev)
    bp = BlendParams(sigma=a.sigma, gamma=1e-4, znear=cam.znear, zfar=cam.zfar)
    d_image = torch.randn((N, H, W, 3), generator=g, device=dev)

    def soft_fused():
        p2f, image = rasterize_softmax(fv, first, num, rs, bp, vc, faces, workspace=ws)
        return rasterize_softmax_backward(fv, first, num, rs, bp, vc, faces, p2f, d_image)[0]

    def soft_unfused():
        p2f, zbuf, bary, dists = rasterize_meshes(fv, first, num, rs, workspace=ws)
        occ = p2f >= 0
        fidx = torch.where(occ, p2f, torch.zeros_like(p2f))
        b = bary.double().requires_grad_(True)
        d = dists.double().requires_grad_(True)
        z = zbuf.double().requires_grad_(True)
        col = (b.unsqueeze(-1) * vc[faces[fidx]]).sum(-2)  # interpolate_face_attributes
        zc = z.clamp(bp.znear, bp.zfar)
        zinv = torch.where(occ, (bp.zfar - zc) / (bp.zfar - bp.znear), torch.full_like(zc, -1.0))
        zmax = zinv.max(-1, keepdim=True).values
        prob = torch.sigmoid(-d / bp.sigma)
        w = torch.where(occ, prob * torch.exp((zinv - zmax) / bp.gamma), torch.zeros_like(prob))
        img = (w.unsqueeze(-1) * col).sum(-2) / w.sum(-1, keepdim=True).clamp_min(1e-300)
        gz, gb, gdd = torch.autograd.grad(img, (z, b, d), d_image.double())
        return rasterize_meshes_backward(fv, first, num, rs, p2f, bary, gz.float(), gb.float(), gdd.float())

    gf, gu = fused(), unfused()
    err = float((gf - gu).abs().max() / gu.abs().max())
    sf, su = soft_fused(), soft_unfused()
    serr = float((sf - su).abs().max() / su.abs().max())
    out = {"config": a.config, "sigma": a.sigma,
           "fused_ms": timed(fused, a.steps, a.warmup), "unfused_ms": timed(unfused, a.steps, a.warmup),
           "fragments_ms": timed(fragments, a.steps, a.warmup), "fused_vs_unfused_grad_rel_err": err,
           "softmax_fused_ms": timed(soft_fused, a.steps, a.warmup),
           "softmax_unfused_ms": timed(soft_unfused, a.steps, a.warmup), "softmax_grad_rel_err": serr}
    from paper_2007_08501_b200 import KernelTimer

    for name, fn in (("fused_kernels_ms", fused), ("softmax_fused_kernels_ms", soft_fused),
                     ("fragments_kernels_ms", fragments)):
        torch.cuda.synchronize()
        with KernelTimer() as kt:
            for _ in range(a.steps):
                fn()
            torch.cuda.synchronize()
        per = {}
        for k, ms in kt.records:
            per[k] = per.get(k, 0.0) + ms / a.steps
        out[name] = per
    out["speedup"] = out["unfused_ms"] / out["fused_ms"]
    out["softmax_speedup"] = out["softmax_unfused_ms"] / out["softmax_fused_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
