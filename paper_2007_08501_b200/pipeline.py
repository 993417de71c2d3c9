"""End-to-end host path: rasterize_meshes forward + backward from pinned HOST buffers, streamed over groups of
meshes so PCIe copies overlap the kernels.

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

import numpy as np
import torch

from .raster import RasterSettings, rasterize_meshes, rasterize_meshes_backward, workspace_bytes


def contiguous_groups(num_faces_per_mesh, n_groups: int) -> list:
    """Split meshes 0..N-1 into <= n_groups contiguous runs of roughly equal face count."""
    counts = np.asarray(num_faces_per_mesh, dtype=np.int64)
    n = len(counts)
    n_groups = max(1, min(n_groups, n))
    target = counts.sum() / n_groups
    groups, start, acc = [], 0, 0
    for b in range(n):
        acc += counts[b]
        if (acc >= target * (len(groups) + 1) and len(groups) < n_groups - 1) or b == n - 1:
            groups.append((start, b + 1))
            start = b + 1
    return [g for g in groups if g[1] > g[0]]


class HostPipeline:
    """Streams forward (+ backward) of a fixed batch layout between pinned host buffers and the GPU."""

    def __init__(self, first, num, settings: RasterSettings, num_faces: int, device, n_groups: int = 8,
                 backward: bool = True):
        self.first = np.asarray(first, dtype=np.int64)
        self.num = np.asarray(num, dtype=np.int64)
        order = np.argsort(self.first, kind="stable")
        if not np.array_equal(order, np.arange(len(order))) or np.any(self.first[1:] < self.first[:-1] + self.num[:-1]):
            raise ValueError("HostPipeline needs packed, ordered, non-overlapping mesh ranges")
        self.s = settings
        self.F = int(num_faces)
        self.N = len(self.num)
        self.dev = torch.device(device)
        self.backward = backward
        H, W = settings.hw
        K = settings.faces_per_pixel
        self.groups = contiguous_groups(self.num, n_groups)
        d = self.dev
        self.fv = torch.empty((self.F, 3, 3), dtype=torch.float64, device=d)
        self.p2f = torch.empty((self.N, H, W, K), dtype=torch.int64, device=d)
        self.zbuf = torch.empty((self.N, H, W, K), dtype=torch.float32, device=d)
        self.bary = torch.empty((self.N, H, W, K, 3), dtype=torch.float32, device=d)
        self.dists = torch.empty((self.N, H, W, K), dtype=torch.float32, device=d)
        if backward:
            self.dz = torch.empty_like(self.zbuf)
            self.db = torch.empty_like(self.bary)
            self.dd = torch.empty_like(self.dists)
            self.grad = torch.zeros((self.F, 3, 3), dtype=torch.float64, device=d)
        ws = max(workspace_bytes(g1 - g0, self.F, settings) for g0, g1 in self.groups)
        self.ws = torch.empty(ws, dtype=torch.uint8, device=d)
        self.g_first = [torch.as_tensor(self.first[g0:g1], device=d) for g0, g1 in self.groups]
        self.g_num = [torch.as_tensor(self.num[g0:g1], device=d) for g0, g1 in self.groups]
        self.g_host = [(self.first[g0:g1].copy(), self.num[g0:g1].copy()) for g0, g1 in self.groups]
        self.h2d, self.comp, self.d2h = (torch.cuda.Stream(device=d) for _ in range(3))

    def face_range(self, g0, g1):
        lo = int(self.first[g0])
        hi = int(self.first[g1 - 1] + self.num[g1 - 1])
        return lo, hi

    def run(self, fv_h, out_h, cot_h=None, grad_h=None):
        """fv_h [F,3,3] f64 pinned; out_h = (p2f, zbuf, bary, dists) pinned host tensors; cot_h = (dz, db, dd)
        pinned fp32; grad_h [F,3,3] f64 pinned. Enqueues everything; the caller synchronises."""
        main = torch.cuda.current_stream(self.dev)
        for st in (self.h2d, self.comp, self.d2h):
            st.wait_stream(main)
        # all host->device copies are enqueued first (one event per group); the compute stream consumes them in
        # order and the device->host stream drains each group as soon as its kernels are done. The *_hr entry
        # points take host copies of the mesh ranges, so no call synchronises and the host runs ahead.
        ev_in = []
        for g0, g1 in self.groups:
            lo, hi = self.face_range(g0, g1)
            with torch.cuda.stream(self.h2d):
                self.fv[lo:hi].copy_(fv_h[lo:hi], non_blocking=True)
                if self.backward:
                    for d, h in zip((self.dz, self.db, self.dd), cot_h):
                        d[g0:g1].copy_(h[g0:g1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.h2d)
                ev_in.append(ev)
        for gi, (g0, g1) in enumerate(self.groups):
            lo, hi = self.face_range(g0, g1)
            self.comp.wait_event(ev_in[gi])
            with torch.cuda.stream(self.comp):
                outs = (self.p2f[g0:g1], self.zbuf[g0:g1], self.bary[g0:g1], self.dists[g0:g1])
                rasterize_meshes(self.fv, self.g_first[gi], self.g_num[gi], self.s, workspace=self.ws, out=outs,
                                 host_ranges=self.g_host[gi])
                ev_fwd = torch.cuda.Event()
                ev_fwd.record(self.comp)
                if self.backward:
                    rasterize_meshes_backward(self.fv, self.g_first[gi], self.g_num[gi], self.s, outs[0], outs[2],
                                              self.dz[g0:g1], self.db[g0:g1], self.dd[g0:g1], out=self.grad,
                                              host_ranges=self.g_host[gi])
                ev_out = torch.cuda.Event()
                ev_out.record(self.comp)
            self.d2h.wait_event(ev_fwd)
            with torch.cuda.stream(self.d2h):
                for h, d in zip(out_h, outs):
                    h[g0:g1].copy_(d, non_blocking=True)
            if self.backward:
                self.d2h.wait_event(ev_out)
                with torch.cuda.stream(self.d2h):
                    grad_h[lo:hi].copy_(self.grad[lo:hi], non_blocking=True)
        for st in (self.h2d, self.comp, self.d2h):
            main.wait_stream(st)
