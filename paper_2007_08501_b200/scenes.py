"""Synthetic scene generators and the host-side camera transform.

Bit-exact numpy restatements of the reference's input side, so the bench and the tests can build the
configs of BASELINE.json on a box without /root/reference:

* ``Rng``                splitmix64 + hand-rolled distributions   (core.hpp:155-185)
* ``axis_angle``         rotation matrix                          (core.cpp:5-19)
* ``ico_sphere``         midpoint-subdivided icosahedron          (templates.cpp:10-58)
* ``cube``               n x n quads per side                     (templates.cpp:60-94)
* ``synthetic_batch``    template ladder batch                    (templates.cpp:96-133)
* ``Camera`` / ``world_to_ndc`` / ``world_to_ndc_backward``       (camera.hpp:19-61, camera.cpp:36-102)
* ``face_verts``         world_to_ndc gathered per face vertex -> the north-star ``face_verts`` [F,3,3]

Every floating-point expression keeps the reference's evaluation order (numpy ufuncs never contract
to FMA), so e.g. ``ico_sphere(3)`` matches ``dr::ico_sphere(3)`` bit for bit; tests/test_scenes.py
checks that against the reference library.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_M64 = (1 << 64) - 1


class Rng:
    """splitmix64 with the reference's hand-rolled distributions (core.hpp:155-185)."""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = float(self.next_u64() >> 11) * 2.0**-53
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def uniform_int(self, n: int) -> int:
        return self.next_u64() % n

    def normal(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        if u1 < 1e-300:
            u1 = 1e-300
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)

    def normal_vec3(self) -> tuple[float, float, float]:
        a = self.normal()
        b = self.normal()
        c = self.normal()
        return (a, b, c)


def _normalized(v):
    x, y, z = v
    n = math.sqrt(x * x + y * y + z * z)
    return (x / n, y / n, z / n) if n > 0 else (0.0, 0.0, 0.0)


def axis_angle(axis, angle: float) -> np.ndarray:
    """Rotation about ``axis`` (core.cpp:5-19); row-major 3x3."""
    ux, uy, uz = _normalized(axis)
    c, s = math.cos(angle), math.sin(angle)
    t = 1 - c
    return np.array(
        [
            [c + ux * ux * t, ux * uy * t - uz * s, ux * uz * t + uy * s],
            [uy * ux * t + uz * s, c + uy * uy * t, uy * uz * t - ux * s],
            [uz * ux * t - uy * s, uz * uy * t + ux * s, c + uz * uz * t],
        ],
        dtype=np.float64,
    )


def mat_apply(m: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """Mat3::apply row by row, left to right (core.hpp:113-117)."""
    x, y, z = pts[:, 0], pts[:, 1], pts[:, 2]
    out = np.empty_like(pts)
    for r in range(3):
        out[:, r] = m[r, 0] * x + m[r, 1] * y + m[r, 2] * z
    return out


def mat_apply_transposed(m: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """Mat3::apply_transposed (core.hpp:118-122)."""
    x, y, z = pts[:, 0], pts[:, 1], pts[:, 2]
    out = np.empty_like(pts)
    for r in range(3):
        out[:, r] = m[0, r] * x + m[1, r] * y + m[2, r] * z
    return out


# --------------------------------------------------------------------------------------------
# meshes


@dataclass
class Meshes:
    """A heterogeneous batch in list form: per-mesh verts [V_b,3] f64 and LOCAL faces [F_b,3] i64."""

    verts: list = field(default_factory=list)
    faces: list = field(default_factory=list)

    def __len__(self):
        return len(self.verts)

    def extend(self, other: "Meshes") -> "Meshes":
        self.verts += other.verts
        self.faces += other.faces
        return self

    def num_faces_per_mesh(self) -> np.ndarray:
        return np.array([len(f) for f in self.faces], dtype=np.int64)

    def num_verts_per_mesh(self) -> np.ndarray:
        return np.array([len(v) for v in self.verts], dtype=np.int64)

    def mesh_to_face_first_idx(self) -> np.ndarray:
        n = self.num_faces_per_mesh()
        return np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)

    def verts_packed(self) -> np.ndarray:
        return np.concatenate(self.verts).astype(np.float64) if self.verts else np.zeros((0, 3))

    def faces_packed(self) -> np.ndarray:
        """Packed faces with GLOBAL vertex indices (batching.cpp:33-43)."""
        out, off = [], 0
        for v, f in zip(self.verts, self.faces):
            out.append(np.asarray(f, dtype=np.int64).reshape(-1, 3) + off)
            off += len(v)
        return np.concatenate(out) if out else np.zeros((0, 3), dtype=np.int64)

    def faces_local_packed(self) -> np.ndarray:
        return (np.concatenate([np.asarray(f, dtype=np.int64).reshape(-1, 3) for f in self.faces])
                if self.faces else np.zeros((0, 3), dtype=np.int64))


_PHI = (1.0 + math.sqrt(5.0)) / 2.0
_ICO_V = [(-1, _PHI, 0), (1, _PHI, 0), (-1, -_PHI, 0), (1, -_PHI, 0),
          (0, -1, _PHI), (0, 1, _PHI), (0, -1, -_PHI), (0, 1, -_PHI),
          (_PHI, 0, -1), (_PHI, 0, 1), (-_PHI, 0, -1), (-_PHI, 0, 1)]
_ICO_F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
          (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
          (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
          (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]


def _normalize_rows(v: np.ndarray) -> np.ndarray:
    x, y, z = v[:, 0], v[:, 1], v[:, 2]
    n = np.sqrt(x * x + y * y + z * z)
    return np.stack([x / n, y / n, z / n], axis=1)


def ico_sphere_rounds(rounds: int) -> Meshes:
    """Icosahedron + ``rounds`` midpoint subdivisions (templates.cpp:34-57), vectorised.

    Midpoint vertex ids are assigned in first-encounter order over faces and their (ab, bc, ca) edges,
    exactly like the reference's std::map-backed ``mid`` lambda.
    """
    verts = _normalize_rows(np.array(_ICO_V, dtype=np.float64))
    faces = np.array(_ICO_F, dtype=np.int64)
    for _ in range(rounds):
        a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
        e0 = np.stack([a, b, c], axis=1).reshape(-1)  # edge starts in visiting order
        e1 = np.stack([b, c, a], axis=1).reshape(-1)
        lo, hi = np.minimum(e0, e1), np.maximum(e0, e1)
        key = lo * (len(verts) + 1) + hi
        uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")
        rank = np.empty_like(order)
        rank[order] = np.arange(len(order))
        mid_id = len(verts) + rank[inv]
        fe0, fe1 = e0[first[order]], e1[first[order]]  # the (a, b) seen at first encounter
        m = (verts[fe0] + verts[fe1]) * 0.5
        verts = np.concatenate([verts, _normalize_rows(m)])
        mid_id = mid_id.reshape(-1, 3)
        ab, bc, ca = mid_id[:, 0], mid_id[:, 1], mid_id[:, 2]
        faces = np.stack([
            np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
            np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], axis=1).reshape(-1, 3)
    return Meshes([verts], [faces])


def ico_sphere(level: int) -> Meshes:
    """dr::ico_sphere(level): level 0 = icosahedron, else level+1 rounds (templates.cpp:24-34)."""
    if level < 0 or level > 6:
        raise ValueError(f"ico_sphere: level {level} outside [0, 6]")
    return ico_sphere_rounds(0 if level == 0 else level + 1)


def cube(half: float = 1.0, n: int = 1) -> Meshes:
    """dr::cube(half, n): 6 sides x n x n quads x 2 triangles (templates.cpp:60-94)."""
    s = 2.0 * half / n
    sides = [
        ((-half, -half, half), (s, 0, 0), (0, s, 0)),
        ((half, -half, -half), (-s, 0, 0), (0, s, 0)),
        ((half, -half, half), (0, 0, -s), (0, s, 0)),
        ((-half, -half, -half), (0, 0, s), (0, s, 0)),
        ((-half, half, half), (s, 0, 0), (0, 0, -s)),
        ((-half, -half, -half), (s, 0, 0), (0, 0, s)),
    ]
    ii, jj = np.meshgrid(np.arange(n + 1, dtype=np.float64), np.arange(n + 1, dtype=np.float64),
                         indexing="ij")
    ii, jj = ii.reshape(-1), jj.reshape(-1)
    vs, fs = [], []
    gi, gj = np.meshgrid(np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64), indexing="ij")
    gi, gj = gi.reshape(-1), gj.reshape(-1)
    for k, (o, du, dv) in enumerate(sides):
        base = k * (n + 1) * (n + 1)
        v = np.stack([(o[c] + du[c] * jj) + dv[c] * ii for c in range(3)], axis=1)
        vs.append(v)
        v00 = base + gi * (n + 1) + gj
        v01, v10 = v00 + 1, v00 + (n + 1)
        v11 = v10 + 1
        fs.append(np.stack([np.stack([v00, v01, v11], 1), np.stack([v00, v11, v10], 1)], 1).reshape(-1, 3))
    return Meshes([np.concatenate(vs)], [np.concatenate(fs)])


def synthetic_batch(mean_faces: float, sigma: float, batch_size: int, seed: int) -> Meshes:
    """dr::synthetic_batch (templates.cpp:96-133)."""
    ladder = [(20, 0, 0)]
    for lvl in range(1, 5):
        ladder.append((20 * (1 << (2 * (lvl + 1))), 0, lvl))
    for n in (1, 2, 3, 4, 6, 8, 12, 16, 24, 32):
        ladder.append((12 * n * n, 1, n))
    ladder.sort(key=lambda e: e[0])  # std::sort by face count; counts are distinct

    def closest(target):
        best = ladder[0]
        for e in ladder:
            if abs(float(e[0]) - target) < abs(float(best[0]) - target):
                best = e
        return best

    rng = Rng(seed)
    hw = math.sqrt(3.0) * sigma
    homogeneous = closest(mean_faces)
    out = Meshes()
    for _ in range(batch_size):
        e = homogeneous if sigma == 0 else closest(rng.uniform(mean_faces - hw, mean_faces + hw))
        out.extend(ico_sphere(e[2]) if e[1] == 0 else cube(1.0, e[2]))
    return out


# --------------------------------------------------------------------------------------------
# camera


@dataclass
class Camera:
    """dr::Camera (camera.hpp:19-35); rotation/translation are world -> view."""

    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: tuple = (0.0, 0.0, 0.0)
    perspective: bool = True
    focal_length: float = 1.0
    principal_point: tuple = (0.0, 0.0)
    ortho_scale: tuple = (1.0, 1.0)
    znear: float = 0.1
    zfar: float = 100.0

    @staticmethod
    def look_from_distance(d: float, perspective: bool = True, focal: float = 1.0) -> "Camera":
        """camera.cpp:27-33: identity rotation, scene pushed to view depth d."""
        return Camera(translation=(0.0, 0.0, float(d)), perspective=perspective,
                      focal_length=float(focal) if perspective else 1.0)

    def packed(self) -> np.ndarray:
        """Flat [kind, R(9), t(3), f, ppx, ppy, sx, sy, znear, zfar] used by the oracle shim."""
        return np.array([1.0 if self.perspective else 0.0, *np.asarray(self.rotation, np.float64).reshape(-1),
                         *self.translation, self.focal_length, *self.principal_point, *self.ortho_scale,
                         self.znear, self.zfar], dtype=np.float64)


def world_to_view(cam: Camera, pts: np.ndarray) -> np.ndarray:
    v = mat_apply(np.asarray(cam.rotation, np.float64), pts)
    t = cam.translation
    return np.stack([v[:, 0] + t[0], v[:, 1] + t[1], v[:, 2] + t[2]], axis=1)


def world_to_ndc(cam: Camera, pts: np.ndarray):
    """camera.cpp:36-70 -> (xy [V,2], z_view [V], clipped [V] bool)."""
    pv = world_to_view(cam, np.asarray(pts, np.float64))
    z = pv[:, 2].copy()
    if cam.perspective:
        clipped = z <= 0
        safe = np.where(clipped, 1.0, z)
        f = cam.focal_length
        x = (f * pv[:, 0]) / safe + cam.principal_point[0]
        y = (f * pv[:, 1]) / safe + cam.principal_point[1]
        x[clipped] = 0.0
        y[clipped] = 0.0
    else:
        clipped = np.zeros(len(z), dtype=bool)
        x = cam.ortho_scale[0] * pv[:, 0]
        y = cam.ortho_scale[1] * pv[:, 1]
    return np.stack([x, y], axis=1), z, clipped


def world_to_ndc_backward(cam: Camera, pts: np.ndarray, d_xy: np.ndarray, d_z: np.ndarray) -> np.ndarray:
    """camera.cpp:72-85, vectorised; clipped points get zero gradient."""
    pv = world_to_view(cam, np.asarray(pts, np.float64))
    if cam.perspective:
        f = cam.focal_length
        z = pv[:, 2]
        ok = z > 0
        zs = np.where(ok, z, 1.0)
        dvx = d_xy[:, 0] * f / zs
        dvy = d_xy[:, 1] * f / zs
        dvz = -f * (d_xy[:, 0] * pv[:, 0] + d_xy[:, 1] * pv[:, 1]) / (zs * zs) + d_z
        dv = np.stack([dvx, dvy, dvz], 1)
        dv[~ok] = 0.0
    else:
        dv = np.stack([d_xy[:, 0] * cam.ortho_scale[0], d_xy[:, 1] * cam.ortho_scale[1], d_z], 1)
    out = mat_apply_transposed(np.asarray(cam.rotation, np.float64), dv)
    if cam.perspective:
        out[~ok] = 0.0
    return out


def face_verts(meshes: Meshes, cam: Camera) -> np.ndarray:
    """north-star input: [F,3,3] (x_ndc, y_ndc, z_view) per face vertex (MR:100-122 gather)."""
    xy, z, _ = world_to_ndc(cam, meshes.verts_packed())
    fp = meshes.faces_packed()
    per_vert = np.concatenate([xy, z[:, None]], axis=1)
    return np.ascontiguousarray(per_vert[fp])  # [F,3,3]


def scatter_face_grads(meshes: Meshes, cam: Camera, grad_face_verts: np.ndarray) -> np.ndarray:
    """grad wrt (x_ndc,y_ndc,z_view) per face vertex -> world-space d_verts [V,3] (MR:380-401)."""
    fp = meshes.faces_packed()
    V = sum(len(v) for v in meshes.verts)
    acc = np.zeros((V, 3), dtype=np.float64)
    np.add.at(acc, fp.reshape(-1), grad_face_verts.reshape(-1, 3))
    return world_to_ndc_backward(cam, meshes.verts_packed(), acc[:, :2], acc[:, 2])


# --------------------------------------------------------------------------------------------
# BASELINE.json configs


def rotated_cubes(seed: int, count: int, fixed_n: int | None = None, draw_faces=(1000.0, 200000.0)) -> Meshes:
    """C4 (seed 4, F~U(1000,200000)) and C5 (seed 5, fixed n=65): cube(0.8, n) rotated by
    axis_angle(rng.normal_vec3(), rng.uniform(0, 2pi)), draws in that order per mesh."""
    rng = Rng(seed)
    out = Meshes()
    for _ in range(count):
        if fixed_n is None:
            f = rng.uniform(*draw_faces)
            n = max(1, int(math.floor(math.sqrt(f / 12.0) + 0.5)))  # std::lround for positive values
        else:
            n = fixed_n
        axis = rng.normal_vec3()
        angle = rng.uniform(0.0, 2.0 * math.pi)
        m = cube(0.8, n)
        out.verts.append(mat_apply(axis_angle(axis, angle), m.verts[0]))
        out.faces.append(m.faces[0])
    return out


def random_soup(rng: Rng, batch: int, max_faces: int, max_extra_verts: int = 20) -> Meshes:
    """test_raster.cpp:113-125 (max_extra_verts=20) / test_acceptance.cpp:149-161 (25, faces 60)."""
    out = Meshes()
    for _ in range(batch):
        nv = 6 + rng.uniform_int(max_extra_verts)
        v = np.empty((nv, 3))
        for i in range(nv):
            a, b, c = rng.normal_vec3()
            v[i] = (a * 0.6, b * 0.6, c * 0.6)
        nf = 1 + rng.uniform_int(max_faces)
        f = np.empty((nf, 3), dtype=np.int64)
        for i in range(nf):
            f[i, 0] = rng.uniform_int(nv)
            f[i, 1] = rng.uniform_int(nv)
            f[i, 2] = rng.uniform_int(nv)
        out.verts.append(v)
        out.faces.append(f)
    return out


CONFIGS = {
    "C1": dict(desc="ico_sphere(3) 5,120 f, 64x64, K=1, blur 0, fwd only", image=64, K=1, blur=0.0, bin_size=16,
               backward=False),
    "C2": dict(desc="synthetic_batch(11000, 18000/(2*sqrt3), 8, seed 0) 83,712 f, 128x128, K=8, blur 1e-4",
               image=128, K=8, blur=1e-4, bin_size=16, backward=True),
    "C3": dict(desc="icosahedron + 8 midpoint rounds 1,310,720 f, 512x512, K=1, blur 0, bin 32", image=512, K=1,
               blur=0.0, bin_size=32, backward=False),
    "C4": dict(desc="64 rotated cubes (Rng 4) 6,581,760 f, 512x512, K=8, blur 1e-4, perspective_correct, "
                    "cull_backfaces", image=512, K=8, blur=1e-4, bin_size=16, backward=True,
               perspective_correct=True, cull_backfaces=True),
    "C5": dict(desc="32 rotated cube(0.8,65) (Rng 5) 1,622,400 f, 256x256, K=50, blur ln(1/1e-4-1)*1e-4",
               image=256, K=50, blur=math.log(1.0 / 1e-4 - 1.0) * 1e-4, bin_size=16, backward=True),
}


def random_clouds(rng: Rng, batch: int, max_n: int, scale: float = 1.0) -> list:
    """tests/helpers.hpp:23-33 (random_cloud_list): per cloud 1 + uniform_int(max_n) points ~ normal_vec3 * scale."""
    out = []
    for _ in range(batch):
        n = 1 + rng.uniform_int(max_n)
        out.append(np.array([np.array(rng.normal_vec3()) * scale for _ in range(n)], np.float64).reshape(n, 3))
    return out


def points_ndc(points: np.ndarray, cam: Camera) -> np.ndarray:
    """world_to_ndc of packed points -> [P,3] (x_ndc, y_ndc, z_view), the point rasterizer's boundary input."""
    xy, z, _ = world_to_ndc(cam, points)
    return np.concatenate([xy, z[:, None]], axis=1)


def config_meshes(name: str) -> Meshes:
    if name == "C1":
        return ico_sphere(3)
    if name == "C2":
        return synthetic_batch(11000.0, 18000.0 / (2.0 * math.sqrt(3.0)), 8, 0)
    if name == "C3":
        return ico_sphere_rounds(8)
    if name == "C4":
        return rotated_cubes(4, 64)
    if name == "C5":
        return rotated_cubes(5, 32, fixed_n=65)
    raise KeyError(name)


def bench_camera() -> Camera:
    """pipeline.cpp:352: look_from_distance(3.0, Perspective, 2.0)."""
    return Camera.look_from_distance(3.0, True, 2.0)
