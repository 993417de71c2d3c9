# A/B ONLY: the round-1 Python HostPipeline (torch streams), kept to compare against the native one (tools/e2e_native_ab.py)
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

from paper_2007_08501_b200.raster import RasterSettings, rasterize_meshes, rasterize_meshes_backward, workspace_bytes


def contiguous_groups(costs, n_groups: int, ramp: int = 0) -> list:
    """Split items 0..N-1 into <= n_groups contiguous runs of roughly equal total cost. ``ramp`` > 0 makes the
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
    """Streams forward (+ backward) of a fixed batch layout between pinned host buffers and the GPU."""

    def __init__(self, first, num, settings: RasterSettings, num_faces: int, device, n_groups: int = 8,
                 backward: bool = True, ramp: int = 2, lookahead: int = 3):
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
        self.lookahead = int(lookahead)  # 0: every H2D enqueued at once
        # instead of an H2D copy of every slot's cotangents
        H, W = settings.hw
        K = settings.faces_per_pixel
        # groups balance PCIe bytes (the e2e bound), not faces: a mesh's slots cost as much as ~0.5M faces
        self.groups = contiguous_groups(transfer_costs(self.num, H * W * K, backward), n_groups, ramp)
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
        # per group: H2D on h2d, kernels on comp, D2H on d2h. The device->host direction carries more bytes than
        # the host->device one (fragments 28 B/slot vs cotangents 20 B/slot), and the two directions share the
        # link's bidirectional budget: group g's H2D waits for the D2H of group g - lookahead, so the inputs arrive
        # just in time instead of taking half the link while the outputs queue. The *_hr entry points take host
        # copies of the mesh ranges, so no call synchronises and the host runs ahead.
        ev_d2h = []
        for gi, (g0, g1) in enumerate(self.groups):
            lo, hi = self.face_range(g0, g1)
            if self.lookahead > 0 and gi >= self.lookahead:
                self.h2d.wait_event(ev_d2h[gi - self.lookahead])
            with torch.cuda.stream(self.h2d):
                self.fv[lo:hi].copy_(fv_h[lo:hi], non_blocking=True)
                if self.backward:
                    for d, h in zip((self.dz, self.db, self.dd), cot_h):
                        d[g0:g1].copy_(h[g0:g1], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(self.h2d)
            self.comp.wait_event(ev_in)
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
            ev = torch.cuda.Event()
            ev.record(self.d2h)
            ev_d2h.append(ev)
        for st in (self.h2d, self.comp, self.d2h):
            main.wait_stream(st)
