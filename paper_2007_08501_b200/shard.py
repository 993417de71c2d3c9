"""Mesh sharding across GPUs (include/dr_shard.h).

Meshes are independent units of the path: each owns one [H,W,K] fragment block and a face range, and nothing is
exchanged between meshes (mesh_raster.cpp:240-283 processes them one after another, :380-401 scatters per face
range). A rank therefore rasterizes its meshes by passing their GLOBAL face ranges of the whole packed batch to
the ordinary entry points: pix_to_face holds global packed face ids and the backward writes only the rank's rows
of grad_face_verts, with no collective on the data path.

The optional gather of the per-mesh outputs to one rank is a list of point-to-point transfers
(``gather_ops`` = dr_shard_gather_ops, computed identically on every rank from the same plan):
  * ``NcclGather``        executes it with NCCL (libdr_shard_b200.so: one ncclGroupStart/End of ncclSend /
                          ncclRecv over NVLink per call, on a caller-chosen stream so it overlaps compute);
  * ``gather_torch``      executes the same list with torch.distributed point-to-point ops (the gloo CPU tests);
  * ``assemble_local``    applies it inside one process (the 1-GPU sharded == unsharded test).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

SEND, RECV, COPY = 0, 1, 2
BUFFERS = ("pix_to_face", "zbuf", "bary", "dists", "grad_face_verts")


class ShardPlan:
    """LPT assignment of meshes to ranks by face count (dr_shard_plan_lpt): owner[m], local_index[m]."""

    def __init__(self, num_faces_per_mesh, world: int):
        costs = np.ascontiguousarray(num_faces_per_mesh, dtype=np.int64)
        self.N, self.world = len(costs), int(world)
        self.owner = np.zeros(self.N, np.int32)
        self.local_index = np.zeros(self.N, np.int32)
        L = _lib.load()
        rc = L.dr_shard_plan_lpt(costs.ctypes.data, self.N, self.world, self.owner.ctypes.data,
                                 self.local_index.ctypes.data)
        if rc:
            raise ValueError(f"dr_shard_plan_lpt: {_lib.last_error()}")

    def meshes(self, rank: int) -> list:
        """Global mesh indices of `rank` in local order."""
        idx = np.nonzero(self.owner == rank)[0]
        return [int(i) for i in idx[np.argsort(self.local_index[idx], kind="stable")]]

    def shards(self) -> list:
        return [self.meshes(r) for r in range(self.world)]


def lpt_partition(costs, world: int) -> list:
    """Sorted mesh index lists per rank (the C-ABI LPT plan)."""
    return ShardPlan(costs, world).shards()


def shard_loads(costs, shards) -> list:
    costs = np.asarray(costs, dtype=np.float64)
    return [float(costs[s].sum()) for s in shards]


def gather_ops(plan: ShardPlan, mesh_first, mesh_num, slots_per_mesh: int, payload_bytes: int, with_grad: bool,
               rank: int, root: int = 0, local_lo: int = 0, local_hi: int = 1 << 30) -> list:
    """dr_shard_gather_ops: the transfers `rank` takes part in, as (kind, peer, buffer name, mesh, src_offset,
    dst_offset, bytes) tuples (byte offsets into the local / global buffers)."""
    L = _lib.load()
    first = np.ascontiguousarray(mesh_first, dtype=np.int64)
    num = np.ascontiguousarray(mesh_num, dtype=np.int64)
    n = C.c_int64(0)
    args = (plan.N, plan.owner.ctypes.data, plan.local_index.ctypes.data, first.ctypes.data, num.ctypes.data,
            int(slots_per_mesh), int(payload_bytes), int(bool(with_grad)), plan.world, int(rank), int(root),
            int(local_lo), int(local_hi))
    rc = L.dr_shard_gather_ops(*args, None, 0, C.byref(n))
    if rc:
        raise ValueError(f"dr_shard_gather_ops: {_lib.last_error()}")
    ops = (_lib.DrShardOp * max(n.value, 1))()
    rc = L.dr_shard_gather_ops(*args, ops, n.value, C.byref(n))
    if rc:
        raise ValueError(f"dr_shard_gather_ops: {_lib.last_error()}")
    return [(o.kind, o.peer, BUFFERS[o.buffer], o.mesh, o.src_offset, o.dst_offset, o.bytes) for o in ops[:n.value]]


def _bytes(t):
    """Flat byte view of a contiguous tensor (writes through it land in the tensor)."""
    import torch

    if not t.is_contiguous():
        raise ValueError("gather buffers must be contiguous")
    return t.reshape(-1).view(torch.uint8)


def gather_torch(ops, local: dict, global_: dict | None):
    """Execute an op list with torch.distributed point-to-point ops (gloo on CPU, or NCCL), all posted before
    any is waited on. ``local`` / ``global_`` map BUFFERS names to tensors (global_ on the root only)."""
    import torch.distributed as dist

    reqs = []
    for kind, peer, buf, _m, src, dst, nb in ops:
        if kind == SEND:
            reqs.append(dist.isend(_bytes(local[buf])[src:src + nb], dst=peer))
        elif kind == RECV:
            reqs.append(dist.irecv(_bytes(global_[buf])[dst:dst + nb], src=peer))
        else:
            g, s_ = _bytes(global_[buf]), _bytes(local[buf])
            if g.data_ptr() + dst != s_.data_ptr() + src:
                g[dst:dst + nb].copy_(s_[src:src + nb])
    for r in reqs:
        r.wait()


def assemble_local(plan: ShardPlan, per_rank: list, global_: dict, mesh_first, mesh_num, slots_per_mesh: int,
                   payload_bytes: int, with_grad: bool, root: int = 0):
    """Apply the gather inside one process: per_rank[r] = rank r's local buffers (dict). The root's receives
    are paired, per sender, with that sender's sends in posting order (the point-to-point matching rule)."""
    recv = [o for o in gather_ops(plan, mesh_first, mesh_num, slots_per_mesh, payload_bytes, with_grad, root, root)]
    for kind, _p, buf, _m, src, dst, nb in recv:
        if kind == COPY:
            g, s_ = _bytes(global_[buf]), _bytes(per_rank[root][buf])
            if g.data_ptr() + dst != s_.data_ptr() + src:
                g[dst:dst + nb].copy_(s_[src:src + nb])
    for r in range(plan.world):
        if r == root:
            continue
        sends = [o for o in gather_ops(plan, mesh_first, mesh_num, slots_per_mesh, payload_bytes, with_grad, r, root)]
        recvs = [o for o in recv if o[0] == RECV and o[1] == r]
        assert len(sends) == len(recvs), (r, len(sends), len(recvs))
        for s, q in zip(sends, recvs):
            assert s[0] == SEND and s[2] == q[2] and s[6] == q[6], (s, q)
            _bytes(global_[q[2]])[q[5]:q[5] + q[6]].copy_(_bytes(per_rank[r][s[2]])[s[4]:s[4] + s[6]])


class NcclGather:
    """The gather over NCCL (libdr_shard_b200.so). The 128-byte NCCL id travels over the default
    torch.distributed group (any backend)."""

    def __init__(self, rank: int, world: int):
        import torch
        import torch.distributed as dist

        self.L = _lib.load_shard()
        self.rank, self.world = rank, world
        buf = C.create_string_buffer(128)
        if rank == 0:
            rc = self.L.dr_shard_unique_id(buf)
            if rc:
                raise RuntimeError(f"dr_shard_unique_id: {self.L.dr_shard_last_error().decode()}")
        obj = [bytes(buf.raw)]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        self.comm = C.c_void_p()
        torch.cuda.current_device()  # the communicator binds to the current device
        rc = self.L.dr_shard_comm_init(world, rank, obj[0], C.byref(self.comm))
        if rc:
            raise RuntimeError(f"dr_shard_comm_init: {self.L.dr_shard_last_error().decode()}")

    @staticmethod
    def buffers(d: dict | None):
        if d is None:
            return None
        return _lib.DrShardBuffers(*[d[n].data_ptr() if d.get(n) is not None else None for n in BUFFERS])

    def gather(self, plan: ShardPlan, mesh_first, mesh_num, slots_per_mesh: int, payload_bytes: int,
               with_grad: bool, local: dict, global_: dict | None, stream, root: int = 0, local_lo: int = 0,
               local_hi: int = 1 << 30):
        first = np.ascontiguousarray(mesh_first, dtype=np.int64)
        num = np.ascontiguousarray(mesh_num, dtype=np.int64)
        lb, gb = self.buffers(local), self.buffers(global_)
        rc = self.L.dr_shard_gather(self.comm, root, plan.N, plan.owner.ctypes.data, plan.local_index.ctypes.data,
                                    first.ctypes.data, num.ctypes.data, int(slots_per_mesh), int(payload_bytes),
                                    int(bool(with_grad)), int(local_lo), int(local_hi), C.byref(lb),
                                    C.byref(gb) if gb is not None else None, C.c_void_p(stream.cuda_stream))
        if rc:
            raise RuntimeError(f"dr_shard_gather: {self.L.dr_shard_last_error().decode()}")

    def close(self):
        if self.comm:
            self.L.dr_shard_comm_destroy(self.comm)
            self.comm = C.c_void_p()
