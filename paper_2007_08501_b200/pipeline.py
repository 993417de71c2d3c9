"""End-to-end host path: rasterize_meshes forward + backward from pinned HOST buffers, streamed over groups of
meshes so PCIe copies overlap the kernels. The pipeline itself is native (csrc/pipeline.cu, dr_host_pipeline_* in
include/dr_raster.h); this module is its Python binding plus the grouping rule restated for the CPU tests.

The reference's rasterize_meshes / rasterize_backward take and return host data (MeshFragments by value,
mesh_raster.hpp:41,66-69). A host caller of the B200 path pays H2D for face_verts (72 B/face) and the
cotangents (20 B/slot fp32) and D2H for the fragments (28 B/slot) and grad_face_verts (72 B/face) — C4: 7.4 GB
per step, far more than the kernels' own time. Meshes are independent (mesh_raster.cpp:240-283), so the batch
is cut into contiguous groups of meshes and run as a three-stream pipeline:

    h2d stream:     copy group g+1's face_verts / cotangents            (overlaps)
    compute stream: rasterize_meshes + rasterize_meshes_backward on g   (overlaps)
    d2h stream:     copy group g-1's fragments / grads back              (overlaps)

Every group's calls use the FULL packed face_verts buffer with the group's global mesh ranges, so face ids are
global and each group's backward writes only its own rows of grad_face_verts (include/dr_raster.h).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .raster import RasterSettings, _check, _ptr


def contiguous_groups(costs, n_groups: int, ramp: int = 0) -> list:
    """(The rule csrc/pipeline.cu applies; tests/test_gpu_parity.py checks the native pipeline's groups against
    it.) Split items 0..N-1 into <= n_groups contiguous runs of roughly equal total cost. ``ramp`` > 0 makes the
    first and last ``ramp`` groups geometrically smaller (1/2, 1/4, ... of a full one): the pipeline's fill (the
    first group's H2D + kernels, before any D2H) and drain (the last group's D2H) then run on small groups."""
    counts = np.asarray(costs, dtype=np.float64)
    n = len(counts)
    n_groups = max(1, min(n_groups, n))
    r = max(0, min(ramp, (n_groups - 1) // 2))
    rel = np.ones(n_groups)
    for i in range(r):
        rel[r - 1 - i] = rel[n_groups - r + i] = 0.5 ** (i + 1)
    bounds = np.cumsum(rel) / rel.sum() * counts.sum()
    groups, start, acc = [], 0, 0.0
    for b in range(n):
        acc += counts[b]
        if (acc >= bounds[len(groups)] - 1e-9 * counts.sum() and len(groups) < n_groups - 1) or b == n - 1:
            groups.append((start, b + 1))
            start = b + 1
    return [g for g in groups if g[1] > g[0]]


def transfer_costs(num_faces_per_mesh, hw_k: int, backward: bool) -> np.ndarray:
    """PCIe bytes per mesh of one e2e step: face_verts in (72 B/face) + fragments out (28 B/slot), and with the
    backward cotangents in (20 B/slot) + grad_face_verts out (72 B/face)."""
    f = np.asarray(num_faces_per_mesh, dtype=np.float64)
    return 72.0 * f * (2 if backward else 1) + (48.0 if backward else 28.0) * hw_k


class HostPipeline:
    """Streams forward (+ backward) of a fixed batch layout between pinned host buffers and the GPU
    (dr_host_pipeline_*: one device allocation, three streams, the caller's stream waits for completion)."""

    def __init__(self, first, num, settings: RasterSettings, num_faces: int, device, n_groups: int = 8,
                 backward: bool = True, ramp: int = 2, lookahead: int = 3):
        self.first = np.ascontiguousarray(first, dtype=np.int64)
        self.num = np.ascontiguousarray(num, dtype=np.int64)
        self.s = settings
        self.F = int(num_faces)
        self.N = len(self.num)
        self.dev = torch.device(device)
        self.backward = backward
        self.L = _lib.load()
        self._c = settings.to_c()
        self.h = C.c_void_p()
        with torch.cuda.device(self.dev):
            rc = self.L.dr_host_pipeline_create(self.first.ctypes.data, self.num.ctypes.data, self.N, self.F,
                                                C.byref(self._c), int(n_groups), int(ramp), int(lookahead),
                                                int(bool(backward)), C.byref(self.h))
        _check(rc, "HostPipeline")
        n = self.L.dr_host_pipeline_groups(self.h, None, 0)
        b = np.zeros(2 * max(n, 1), np.int64)
        self.L.dr_host_pipeline_groups(self.h, b.ctypes.data, n)
        self.groups = [(int(b[2 * g]), int(b[2 * g + 1])) for g in range(n)]

    def run(self, fv_h, out_h, cot_h=None, grad_h=None):
        """fv_h [F,3,3] f64 pinned; out_h = (p2f, zbuf, bary, dists) pinned host tensors; cot_h = (dz, db, dd)
        pinned fp32; grad_h [F,3,3] f64 pinned. Enqueues everything; the current stream waits for completion."""
        H, W = self.s.hw
        K = self.s.faces_per_pixel
        shp = (self.N, H, W, K)
        for t, want, dt in zip(out_h, (shp, shp, shp + (3,), shp), (torch.int64,) + (torch.float32,) * 3):
            if tuple(t.shape) != want or t.dtype != dt or t.is_cuda or not t.is_contiguous():
                raise ValueError(f"HostPipeline.run: host output {tuple(t.shape)} {t.dtype}, want {want} {dt}")
        cz = cb = cd = gr = None
        if self.backward:
            cz, cb, cd = (t.contiguous() for t in cot_h)
            gr = grad_h
        with torch.cuda.device(self.dev):
            st = C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
            rc = self.L.dr_host_pipeline_run(self.h, _ptr(fv_h), *(_ptr(t) for t in out_h), _ptr(cz), _ptr(cb),
                                             _ptr(cd), _ptr(gr), st)
        _check(rc, "HostPipeline.run")

    def close(self):
        if self.h:
            self.L.dr_host_pipeline_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
