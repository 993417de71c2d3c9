"""fit_silhouette on the GPU path: the reference's silhouette-fitting demo
(/root/reference/proj/src/pipeline.cpp:100-205, FitConfig pipeline.hpp:56-78) with every rasterization step on the
B200 kernels and the whole loop device-resident.

Per iteration and view (pipeline.cpp:146-160): world_to_face_verts (camera kernel) -> fused rasterize_meshes +
silhouette_blend (K2 emit mode 1, no fragment payload written) -> silhouette_iou_loss and its backward ->
fused silhouette_blend_backward + rasterize_backward (k_silhouette_backward) -> face_verts_backward (vertex
scatter + world_to_ndc_backward kernels). The regularizers (geometry.cpp:556-649: mean squared edge length, L1
uniform Laplacian) and the Adam update (pipeline.cpp:178-190) are small O(V + E) fp64 tensor ops on the same
stream; the loss trace stays on the device and is read once at the end, so an iteration never synchronises.

The silhouette runs through the fp64 entry points (fp64 alpha and cotangent): Adam divides every coordinate's
step by its own gradient magnitude, so fp32 rounding in near-zero (cancelling) gradient components would turn into
full-size steps of arbitrary sign. Remaining differences from the reference: fp64 sums are tree reductions / atomics
instead of serial loops, and a non-finite total is reported after the loop (the reference throws at that
iteration; the result is the same exception). OBJ input/output (target_path, output_mesh,
output_trace) is file I/O outside the path and not mirrored.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .raster import (RasterSettings, UsageError, face_verts_backward, rasterize_silhouette,
                     rasterize_silhouette_backward, workspace_bytes, world_to_face_verts)
from .scenes import Camera, Meshes, axis_angle, cube, ico_sphere


class NonFiniteError(RuntimeError):
    """dr::NonFiniteError (core.hpp): the fit diverged."""


@dataclass
class FitConfig:
    """pipeline.hpp:56-78 (defaults are the reference's)."""

    target_spec: str = "sphere:2"
    target_scale: float = 1.0
    template_level: int = 2
    num_views: int = 2
    iterations: int = 400
    step_size: float = 0.01
    lambda_laplacian: float = 19.0
    lambda_edge: float = 0.2
    image_size: int = 64
    faces_per_pixel: int = 24
    coarse_blur_radius: float = 4e-3
    coarse_sigma: float = 2e-3
    coarse_fraction: float = 0.6
    blur_radius: float = 1e-4
    sigma: float = 1e-5
    camera_distance: float = 3.0
    focal_length: float = 2.0


@dataclass
class FitTraceRow:
    """pipeline.hpp:80-83."""

    iter: int
    l_s: float
    l_l: float
    l_e: float
    total: float


@dataclass
class FitResult:
    """pipeline.hpp:85-89: the fitted mesh (verts on the device, faces local), the loss trace, and the mean
    silhouette loss of the fitted mesh over the views."""

    verts: torch.Tensor
    faces: np.ndarray
    trace: list = field(default_factory=list)
    final_silhouette_loss: float = 0.0


def mesh_from_spec(spec: str) -> Meshes:
    """pipeline.cpp:20-27: "sphere[:level]" or "cube[:n]"."""
    kind, _, param = spec.partition(":")
    p = int(param) if param else -1
    if kind == "sphere":
        return ico_sphere(2 if p < 0 else p)
    if kind == "cube":
        return cube(1.0, 1 if p < 0 else p)
    raise UsageError(f"unknown template spec '{spec}'")


def view_camera(distance: float, focal: float, perspective: bool, angle: float) -> Camera:
    """pipeline.cpp:35-41: rotate the world about +y by ``angle``, then push it to view depth ``distance``."""
    r = axis_angle((0.0, 1.0, 0.0), angle)
    if perspective:
        return Camera(rotation=r, translation=(0.0, 0.0, float(distance)), perspective=True,
                      focal_length=float(focal))
    return Camera(rotation=r, translation=(0.0, 0.0, float(distance)), perspective=False)


class MeshRegularizers:
    """edge_length_loss / laplacian_loss and their backwards (geometry.cpp:540-649) for a fixed topology, on the
    device. The per-element unique undirected edge lists (element_edges, geometry.cpp:540-552) are built once on
    the host; values and gradients are fp64 tensor ops."""

    def __init__(self, meshes: Meshes, device):
        dev = torch.device(device)
        n = len(meshes)
        vcount = meshes.num_verts_per_mesh()
        voff = np.concatenate([[0], np.cumsum(vcount)[:-1]]).astype(np.int64)
        eu, ev, eel, ecount = [], [], [], np.zeros(n, np.int64)
        for b, f in enumerate(meshes.faces):
            f = np.asarray(f, np.int64).reshape(-1, 3)
            a = np.concatenate([f[:, 0], f[:, 1], f[:, 2]])
            c = np.concatenate([f[:, 1], f[:, 2], f[:, 0]])
            lo, hi = np.minimum(a, c), np.maximum(a, c)
            keep = lo != hi
            e = np.unique(np.stack([lo[keep], hi[keep]], 1), axis=0) if keep.any() else np.zeros((0, 2), np.int64)
            eu.append(e[:, 0] + voff[b])
            ev.append(e[:, 1] + voff[b])
            eel.append(np.full(len(e), b, np.int64))
            ecount[b] = len(e)
            # an element's vertices must all have neighbours (laplacian_loss throws IsolatedVertexError)
            deg = np.bincount(np.concatenate([e[:, 0], e[:, 1]]), minlength=int(vcount[b]))
            if (deg == 0).any():
                raise UsageError(f"vertex {int(np.argmax(deg == 0))} of mesh {b} has no neighbors")
        cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64))
        self.n = n
        self.u = torch.as_tensor(cat(eu), device=dev)
        self.v = torch.as_tensor(cat(ev), device=dev)
        self.edge_el = torch.as_tensor(cat(eel), device=dev)
        self.ecount = torch.as_tensor(ecount, dtype=torch.float64, device=dev)
        self.vert_el = torch.as_tensor(np.repeat(np.arange(n), vcount), device=dev)
        self.vcount = torch.as_tensor(vcount, dtype=torch.float64, device=dev)
        # symmetric adjacency (both directions of every edge) for the uniform Laplacian
        self.rows = torch.cat([self.u, self.v])
        self.cols = torch.cat([self.v, self.u])
        V = int(vcount.sum())
        # neighbour table [V, max_deg] in ascending neighbour order (neighbor_lists sorts, geometry.cpp:590-600),
        # padded with -1: the Laplacian sums neighbours serially in exactly the reference's order, because its
        # L1 subgradient sign(mean - v) is discontinuous at 0 and symmetric meshes hit 0 exactly
        r = torch.cat([self.u, self.v]).cpu().numpy()
        c = torch.cat([self.v, self.u]).cpu().numpy()
        order = np.lexsort((c, r))
        r, c = r[order], c[order]
        deg = np.bincount(r, minlength=V)
        start = np.concatenate([[0], np.cumsum(deg)[:-1]])
        nbr = np.full((V, max(1, int(deg.max()) if V else 1)), -1, np.int64)
        nbr[r, np.arange(len(r)) - start[r]] = c
        self.nbr = torch.as_tensor(nbr, device=dev)
        self.inv_deg = 1.0 / torch.as_tensor(deg, dtype=torch.float64, device=dev)  # mean *= 1.0 / deg
        self.has_edges = self.ecount > 0

    def edge_length_loss(self, verts):
        """geometry.cpp:556-570 -> (per_element [N], mean)."""
        d = verts[self.u] - verts[self.v]
        n2 = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]
        s = torch.zeros(self.n, dtype=torch.float64, device=verts.device).index_add_(0, self.edge_el, n2)
        per = torch.where(self.has_edges, s / self.ecount.clamp_min(1.0), torch.zeros_like(s))
        return per, per.sum() / self.n

    def edge_length_loss_backward(self, verts, d_mean):
        """geometry.cpp:572-588."""
        coeff = (d_mean / self.n * 2.0 / self.ecount.clamp_min(1.0))[self.edge_el]
        g = (verts[self.u] - verts[self.v]) * coeff[:, None]
        out = torch.zeros_like(verts)
        out.index_add_(0, self.u, g)
        out.index_add_(0, self.v, -g)
        return out

    def _lap(self, verts):
        s = torch.zeros_like(verts)
        for j in range(self.nbr.shape[1]):  # serial over the sorted neighbours (+0.0 for the padding is exact)
            col = self.nbr[:, j]
            s = s + torch.where((col >= 0)[:, None], verts[col.clamp_min(0)], torch.zeros((), dtype=verts.dtype,
                                                                                          device=verts.device))
        return s * self.inv_deg[:, None] - verts  # mean - v (geometry.cpp:619-621)

    def laplacian_loss(self, verts):
        """geometry.cpp:606-627 -> (per_element [N], mean)."""
        a = self._lap(verts).abs().sum(1)
        s = torch.zeros(self.n, dtype=torch.float64, device=verts.device).index_add_(0, self.vert_el, a)
        per = s / self.vcount
        return per, per.sum() / self.n

    def laplacian_loss_backward(self, verts, d_mean):
        """geometry.cpp:629-649: L1 subgradient sign(mean - v) (0 at 0)."""
        sg = torch.sign(self._lap(verts))
        coeff = (d_mean / self.n / self.vcount)[self.vert_el]
        out = -sg * coeff[:, None]
        w = sg * (coeff * self.inv_deg)[:, None]
        out.index_add_(0, self.cols, w[self.rows])
        return out


def silhouette_iou_loss(pred, gt):
    """geometry.cpp:651-661 (both all-zero -> 0), as a device scalar."""
    pg = pred * gt
    inter = pg.sum()
    uni = (pred + gt - pg).sum()
    return torch.where(uni > 0, 1.0 - inter / uni, torch.zeros_like(uni))


def silhouette_iou_loss_backward(pred, gt, d_loss=1.0):
    """geometry.cpp:663-682: -d (g U - I (1 - g)) / U^2 (zero when U <= 0)."""
    pg = pred * gt
    inter = pg.sum()
    uni = (pred + gt - pg).sum()
    g = -d_loss * (gt * uni - inter * (1.0 - gt)) / (uni * uni)
    return torch.where(uni > 0, g, torch.zeros_like(g))


class _Views:
    """The fixed cameras + raster settings of one fit; silhouettes of packed verts on the GPU. Every call is
    non-synchronising (host copies of the mesh ranges, the unchecked projection after a one-time index check,
    a preallocated workspace), so an iteration can be captured into a CUDA graph."""

    def __init__(self, cfg: FitConfig, m: Meshes, dev):
        self.cams = [view_camera(cfg.camera_distance, cfg.focal_length, True,
                                 2.0 * 3.14159265358979323846 * v / cfg.num_views) for v in range(cfg.num_views)]
        self.faces = torch.as_tensor(m.faces_packed(), dtype=torch.int64, device=dev)
        self.host = (m.mesh_to_face_first_idx(), m.num_faces_per_mesh())
        self.first, self.num = (torch.as_tensor(x, device=dev) for x in self.host)
        self.V = int(m.num_verts_per_mesh().sum())
        if len(self.faces) and (int(self.faces.min()) < 0 or int(self.faces.max()) >= self.V):
            raise UsageError("face vertex index out of range")
        self.rs = RasterSettings(image_size=cfg.image_size, faces_per_pixel=cfg.faces_per_pixel)
        self.ws = torch.empty(workspace_bytes(len(m), len(self.faces), self.rs), dtype=torch.uint8, device=dev)

    def set_blur(self, blur: float):
        self.rs = RasterSettings(image_size=self.rs.image_size, faces_per_pixel=self.rs.faces_per_pixel,
                                 blur_radius=blur, znear=self.cams[0].znear)
        need = workspace_bytes(len(self.host[0]), len(self.faces), self.rs)
        if need > self.ws.numel():
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.ws.device)

    def alpha(self, verts, v: int, sigma: float, want_p2f: bool):
        fv = world_to_face_verts(verts, self.faces, self.cams[v], check=False)
        p2f, a = rasterize_silhouette(fv, self.first, self.num, self.rs, sigma, want_pix_to_face=want_p2f,
                                      workspace=self.ws, out_dtype=torch.float64, host_ranges=self.host)
        return fv, p2f, a

    def grad(self, verts, v: int, fv, sigma: float, p2f, d_alpha):
        g_fv = rasterize_silhouette_backward(fv, self.first, self.num, self.rs, sigma, p2f, d_alpha,
                                             host_ranges=self.host)
        return face_verts_backward(verts, self.faces, self.cams[v], g_fv)


class _Step:
    """One fit iteration (pipeline.cpp:146-190) on static tensors: reads verts / Adam state / the bias
    corrections c1, c2 (device scalars) / the band's targets, updates verts and the Adam state in place and
    writes (l_s / views, l_l, l_e, total) into ``row``. Device work only, so it can be replayed as a graph."""

    def __init__(self, cfg: FitConfig, views: _Views, reg: MeshRegularizers, verts, targets, sigma):
        self.cfg, self.views, self.reg, self.verts, self.targets, self.sigma = cfg, views, reg, verts, targets, sigma
        dev = verts.device
        self.m = torch.zeros_like(verts)
        self.v = torch.zeros_like(verts)
        self.c1 = torch.ones((), dtype=torch.float64, device=dev)
        self.c2 = torch.ones((), dtype=torch.float64, device=dev)
        self.row = torch.zeros(4, dtype=torch.float64, device=dev)

    def __call__(self):
        cfg, views, reg, verts = self.cfg, self.views, self.reg, self.verts
        b1, b2, adam_eps = 0.9, 0.999, 1e-8
        grad = torch.zeros_like(verts)
        l_s = torch.zeros((), dtype=torch.float64, device=verts.device)
        for v in range(cfg.num_views):
            fv, p2f, alpha = views.alpha(verts, v, self.sigma, True)
            tgt = self.targets[v]
            l_s = l_s + silhouette_iou_loss(alpha, tgt)
            d_alpha = silhouette_iou_loss_backward(alpha, tgt, 1.0)
            grad += views.grad(verts, v, fv, self.sigma, p2f, d_alpha)
        _, l_l = reg.laplacian_loss(verts)
        _, l_e = reg.edge_length_loss(verts)
        total = l_s + cfg.lambda_laplacian * l_l + cfg.lambda_edge * l_e
        grad += reg.laplacian_loss_backward(verts, cfg.lambda_laplacian)
        grad += reg.edge_length_loss_backward(verts, cfg.lambda_edge)
        self.row.copy_(torch.stack([l_s / cfg.num_views, l_l, l_e, total]))
        # pipeline.cpp:182-186, same operation order
        self.m.copy_(b1 * self.m + (1 - b1) * grad)
        self.v.copy_(b2 * self.v + (1 - b2) * grad * grad)
        verts -= cfg.step_size * (self.m / self.c1) / (torch.sqrt(self.v / self.c2) + adam_eps)


def fit_silhouette(cfg: FitConfig, device="cuda", graph: bool = True) -> FitResult:
    """dr::fit_silhouette (pipeline.cpp:100-205) on the B200 path. ``graph``: each band's iteration is captured
    once into a CUDA graph and replayed (one launch per iteration instead of ~150 kernel launches + host work)."""
    if cfg.num_views < 2:
        raise UsageError("fit requires at least 2 views")
    dev = torch.device(device)
    target = mesh_from_spec(cfg.target_spec)
    tverts = torch.as_tensor(target.verts_packed(), device=dev)
    if cfg.target_scale != 1.0:
        tverts = tverts * cfg.target_scale  # scale_mesh, pipeline.cpp:29-33
    tv = _Views(cfg, target, dev)
    mesh = ico_sphere(cfg.template_level)
    views = _Views(cfg, mesh, dev)
    reg = MeshRegularizers(mesh, dev)
    verts = torch.as_tensor(mesh.verts_packed(), device=dev).clone()
    coarse_iters = int(cfg.coarse_fraction * cfg.iterations)
    bands = [(0, coarse_iters, cfg.coarse_sigma, cfg.coarse_blur_radius)] if coarse_iters > 0 else []
    bands.append((coarse_iters if coarse_iters > 0 else 0, cfg.iterations, cfg.sigma, cfg.blur_radius))
    trace = torch.zeros((max(cfg.iterations, 0), 4), dtype=torch.float64, device=dev)
    b1, b2 = 0.9, 0.999
    step = None
    for lo, hi, sigma, blur in bands:
        # pipeline.cpp:119-125 / 167-172: target silhouettes re-rendered per band, Adam restarted
        tv.set_blur(blur)
        views.set_blur(blur)
        targets = [tv.alpha(tverts, v, sigma, False)[2] for v in range(cfg.num_views)]
        step = _Step(cfg, views, reg, verts, targets, sigma)
        run = step
        if graph and dev.type == "cuda" and hi > lo:
            # warm up on a side stream (library loads, allocator), restoring the state it touched
            saved = verts.clone()
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream(dev).wait_stream(side)
            verts.copy_(saved)
            step.m.zero_()
            step.v.zero_()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            run = g.replay
        for k, it in enumerate(range(lo, hi)):
            step.c1.fill_(1.0 - math.pow(b1, k + 1))
            step.c2.fill_(1.0 - math.pow(b2, k + 1))
            run()
            trace[it].copy_(step.row)

    trace_np = trace.cpu().numpy()
    bad = np.nonzero(~np.isfinite(trace_np[:, 3]))[0]
    if len(bad):
        raise NonFiniteError(f"fit diverged at iteration {int(bad[0])}")
    l_s = sum(float(silhouette_iou_loss(views.alpha(verts, v, step.sigma, False)[2], step.targets[v]))
              for v in range(cfg.num_views)) if step is not None else 0.0
    rows = [FitTraceRow(i, *map(float, r)) for i, r in enumerate(trace_np)]
    return FitResult(verts=verts, faces=mesh.faces_local_packed(), trace=rows,
                     final_silhouette_loss=l_s / cfg.num_views)
