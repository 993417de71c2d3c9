"""Whole-batch parity on the headline configs (C4, C5): every mesh, every slot, every gradient element.

The reference's own acceptance standard is whole-output bit-identity over every scene
(/root/reference/proj/tests/test_acceptance.cpp:143-183). Two legs per config:

* reference semantics (the only ones the reference has: no perspective_correct / cull_backfaces): the GPU's fp64
  payload is compared BIT-EXACT with ``dr::rasterize_meshes`` run by the reference library itself
  (oracle/_ref/libdr3d_ref.so, mesh_raster.cpp:234-285) on all meshes, and the GPU backward chained through the
  device vertex scatter + ``world_to_ndc_backward`` with ``dr::rasterize_backward`` (mesh_raster.cpp:287-403)
  element by element;
* the config's own flags (C4: perspective_correct + cull_backfaces): the GPU vs the oracle restatement
  (oracle/raster_oracle.c) on all meshes, one oracle call per mesh on a thread pool (ctypes drops the GIL).
  fp64 payload bit-exact, fp32 payload (the product/bench path) pix_to_face bit-exact and zbuf/bary/dists within
  1e-5 rel / 1e-6 abs, gradients element by element for both payloads.

Gradient criterion (north_star: "face_verts gradients within 1e-4 relative"), per element:
    |got - want| <= GRAD_RTOL * |want| + GRAD_ATOL_SCALE * max|want|
GRAD_ATOL_SCALE = 1e-8: an element whose contributions cancel to below 1e-8 of the largest gradient carries no
relative information at fp32-payload precision. Emulated on the CPU (oracle backward fed fp32-rounded vs fp64
barycentrics, C4 meshes 0/5/40) the absolute term an element actually needs is <= 3e-11 of the scale, so the
bound has 300x headroom while remaining 4 orders tighter than the max-normalised 1e-4 it replaces.

Set DR_PARITY_REPORT=<path> to append one JSON line per check (worst element, counts) to <path>.
"""
from __future__ import annotations

import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from paper_2007_08501_b200 import scenes as S
from tests._common import boundary, fast_cotangents, orc_settings, raster_settings

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RTOL, ATOL = 1e-5, 1e-6
GRAD_RTOL, GRAD_ATOL_SCALE = 1e-4, 1e-8
GROUP = 8  # meshes per reference call (bounds host memory: 8 C4 meshes = 0.8 GB of fp64 fragments)


def _report(**kw):
    path = os.environ.get("DR_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(kw) + "\n")


def grad_check(got, want, what):
    """Per-element |got-want| <= GRAD_RTOL*|want| + GRAD_ATOL_SCALE*max|want|; returns the worst element's stats."""
    got, want = np.asarray(got, np.float64).ravel(), np.asarray(want, np.float64).ravel()
    assert got.shape == want.shape
    scale = float(np.abs(want).max()) if want.size else 0.0
    err = np.abs(got - want)
    bound = GRAD_RTOL * np.abs(want) + GRAD_ATOL_SCALE * scale
    ratio = err / np.maximum(bound, 1e-300)
    i = int(np.argmax(ratio)) if ratio.size else 0
    nz = want != 0
    rel = err[nz] / np.abs(want[nz])
    stats = {"check": what, "elements": int(want.size), "nonzero": int(nz.sum()), "scale": scale,
             "worst_index": i, "worst_got": float(got[i]) if got.size else 0.0,
             "worst_want": float(want[i]) if want.size else 0.0, "worst_err_over_bound": float(ratio[i]) if ratio.size
             else 0.0, "max_rel_err_nonzero": float(rel.max()) if rel.size else 0.0,
             "p99999_rel_err_nonzero": float(np.quantile(rel, 0.99999)) if rel.size else 0.0}
    _report(**stats)
    assert ratio.size == 0 or ratio[i] <= 1.0, f"{what}: worst element {stats}"
    return stats


def _dev(x, cuda):
    return torch.as_tensor(np.ascontiguousarray(x), device=cuda)


def _gpu_fwd(fv, first, num, rs, cuda, out_dtype):
    from paper_2007_08501_b200 import rasterize_meshes

    return rasterize_meshes(_dev(fv, cuda), _dev(first, cuda), _dev(num, cuda), rs, out_dtype=out_dtype)


def _gpu_bwd(fv, first, num, rs, cuda, p2f, bary, dz, db, dd):
    from paper_2007_08501_b200 import rasterize_meshes_backward

    return rasterize_meshes_backward(_dev(fv, cuda), _dev(first, cuda), _dev(num, cuda), rs, p2f, bary, dz, db, dd)


def _groups(n):
    return [list(range(s, min(s + GROUP, n))) for s in range(0, n, GROUP)]


def _subset(m: S.Meshes, idx):
    return S.Meshes([m.verts[i] for i in idx], [m.faces[i] for i in idx])


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_full_config_reference_semantics_vs_reference_library(cfg, reflib, cuda):
    """All meshes at reference semantics: GPU fp64 payload == dr::rasterize_meshes bit for bit; world-space GPU
    gradients (rasterize backward -> device scatter -> world_to_ndc_backward) vs dr::rasterize_backward per
    element, on the reference's own fragments and the same cotangents."""
    from paper_2007_08501_b200 import face_verts_backward

    c = S.CONFIGS[cfg]
    H, K, blur, tile = c["image"], c["K"], c["blur"], c["bin_size"]
    m, cam = S.config_meshes(cfg), S.bench_camera()
    reflib.set_num_threads(os.cpu_count() or 1)
    rs = raster_settings(H, K, blur, cam, bin_size=tile)
    occupied = 0
    for gi, idx in enumerate(_groups(len(m.verts))):
        sub = _subset(m, idx)
        fv, first, num = boundary(sub, cam)
        rb = reflib.batch(sub)
        want = reflib.rasterize(rb, cam.packed(), H, H, K, blur, tile)
        got = [t.cpu().numpy() for t in _gpu_fwd(fv, first, num, rs, cuda, torch.float64)]
        for name, g, w in zip(("pix_to_face", "zbuf", "bary", "dists"), got, want):
            bad = np.argwhere(g != w)
            assert bad.size == 0, f"{cfg} meshes {idx[0]}..{idx[-1]} {name} differs at {bad[:5].tolist()}"
        occupied += int((want[0] >= 0).sum())
        dz, db, dd = fast_cotangents(want[0].size, 100 + gi)
        d_ref = reflib.rasterize_backward(rb, cam.packed(), H, H, K, blur, want, dz, db, dd, tile)
        shp = want[0].shape
        g_fv = _gpu_bwd(fv, first, num, rs, cuda, _dev(want[0], cuda), _dev(want[2], cuda),
                        _dev(dz.reshape(shp), cuda), _dev(db.reshape(shp + (3,)), cuda), _dev(dd.reshape(shp), cuda))
        d_got = face_verts_backward(_dev(sub.verts_packed(), cuda), _dev(sub.faces_packed(), cuda), cam,
                                    g_fv).cpu().numpy()
        grad_check(d_got, d_ref, f"{cfg} ref-semantics d_verts meshes {idx[0]}..{idx[-1]}")
    _report(check=f"{cfg} ref-semantics forward", meshes=len(m.verts), occupied_slots=occupied, bit_exact=True)
    assert occupied > 0


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_full_config_flags_vs_oracle(cfg, oracle, cuda):
    """All meshes with the config's own flags: GPU vs the oracle restatement, one oracle call per mesh on a
    thread pool. fp64 payload bit-exact; fp32 payload p2f bit-exact + payload tolerance; gradients per element for
    the fp64 path (oracle fragments, fp64 cotangents) and the fp32 product path (GPU fp32 fragments and fp32
    cotangents, oracle fed the same fp32-rounded cotangents)."""
    c = S.CONFIGS[cfg]
    H, K, blur, tile = c["image"], c["K"], c["blur"], c["bin_size"]
    persp, cull = bool(c.get("perspective_correct", False)), bool(c.get("cull_backfaces", False))
    m, cam = S.config_meshes(cfg), S.bench_camera()
    fv, first, num = boundary(m, cam)
    N = len(first)
    rs = raster_settings(H, K, blur, cam, persp_correct=persp, cull=cull, bin_size=tile)
    o = orc_settings(H, K, blur, cam, persp_correct=int(persp), cull=int(cull), bin_size=tile)

    p32, z32, b32, d32 = _gpu_fwd(fv, first, num, rs, cuda, torch.float32)

    def oracle_mesh(b):
        # the mesh alone (local face ids 0..n-1): the oracle's gradient buffer is then this mesh's faces only
        sl = slice(int(first[b]), int(first[b] + num[b]))
        fv_b = np.ascontiguousarray(fv[sl])
        fr = oracle.forward(fv_b, [0], num[[b]], o)
        S_ = fr[0].size
        dz, db, dd = (x.astype(np.float32).astype(np.float64) for x in fast_cotangents(S_, 1000 + b))
        g64 = oracle.backward(fv_b, [0], num[[b]], o, fr[0], fr[2], dz, db, dd)
        return b, fv_b, fr, (dz, db, dd), g64

    def results():
        # bounded window of in-flight meshes (C4: ~200 MB of fragments + cotangents each)
        width = os.cpu_count() or 4
        with ThreadPoolExecutor(max_workers=width) as ex:
            futs = [ex.submit(oracle_mesh, b) for b in range(min(width, N))]
            for b in range(N):
                r = futs[b].result()
                futs[b] = None
                if b + width < N:
                    futs.append(ex.submit(oracle_mesh, b + width))
                yield r

    zero = np.zeros(1, np.int64)
    for b, fv_b, fr, (dz, db, dd), g_want in results():
        shp = fr[0].shape
        # fp64 payload bit-exact (GPU, this mesh alone)
        got64 = [t.cpu().numpy() for t in _gpu_fwd(fv_b, zero, num[[b]], rs, cuda, torch.float64)]
        for name, g, w in zip(("pix_to_face", "zbuf", "bary", "dists"), got64, fr):
            bad = np.argwhere(g != w)
            assert bad.size == 0, f"{cfg} mesh {b} fp64 {name} differs at {bad[:5].tolist()}"
        # fp32 payload of the whole-batch call (global face ids): p2f bit-exact, payload within tolerance
        p, z, ba, di = (t[b:b + 1].cpu().numpy() for t in (p32, z32, b32, d32))
        p_want = np.where(fr[0] >= 0, fr[0] + first[b], -1)
        assert np.array_equal(p, p_want), f"{cfg} mesh {b} fp32 pix_to_face differs"
        for name, g, w in (("zbuf", z, fr[1]), ("bary", ba, fr[2]), ("dists", di, fr[3])):
            np.testing.assert_allclose(g.astype(np.float64), w, rtol=RTOL, atol=ATOL,
                                       err_msg=f"{cfg} mesh {b} fp32 {name}")
        # backward, fp64 path on the oracle's fragments
        t64 = lambda a, s: torch.as_tensor(np.ascontiguousarray(a).reshape(s), device=cuda)  # noqa: E731
        g_got = _gpu_bwd(fv_b, zero, num[[b]], rs, cuda, t64(fr[0], shp), t64(fr[2], shp + (3,)),
                         t64(dz, shp), t64(db, shp + (3,)), t64(dd, shp)).cpu().numpy()
        grad_check(g_got, g_want, f"{cfg} flags fp64 grad mesh {b}")
        # backward, fp32 product path: the whole-batch call's fp32 fragments (shifted to local ids) + fp32
        # cotangents
        t32 = lambda a, s: torch.as_tensor(a.reshape(s), dtype=torch.float32, device=cuda)  # noqa: E731
        p_loc = torch.where(p32[b:b + 1] >= 0, p32[b:b + 1] - int(first[b]), p32[b:b + 1]).contiguous()
        g_got32 = _gpu_bwd(fv_b, zero, num[[b]], rs, cuda, p_loc, b32[b:b + 1].contiguous(), t32(dz, shp),
                           t32(db, shp + (3,)), t32(dd, shp)).cpu().numpy()
        grad_check(g_got32, g_want, f"{cfg} flags fp32 grad mesh {b}")
    _report(check=f"{cfg} flags forward", meshes=N, bit_exact_fp64=True)
