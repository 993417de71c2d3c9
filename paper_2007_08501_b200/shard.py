"""Mesh sharding across GPUs.

Meshes are independent units of the path: each owns one [H,W,K] fragment block and a disjoint face range,
and nothing is exchanged between meshes (mesh_raster.cpp:240-283 processes them one after another). A batch
therefore shards by mesh with no collective on the data path; ``lpt_partition`` balances ranks by face count
(longest-processing-time greedy). ``gather_fragments`` is the optional output gather to one rank
(NCCL point-to-point over NVLink when the process group is NCCL; gloo in the CPU tests).
"""
from __future__ import annotations

import heapq

import numpy as np


def lpt_partition(costs, world: int) -> list:
    """Assign items to `world` bins, largest cost first to the least-loaded bin. Returns sorted index lists
    (ties broken by rank then index, so the result is deterministic)."""
    costs = np.asarray(costs, dtype=np.float64)
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(x) for x in out]


def shard_loads(costs, shards) -> list:
    costs = np.asarray(costs, dtype=np.float64)
    return [float(costs[s].sum()) for s in shards]


def globalize_face_ids(pix_to_face, local_first, global_first):
    """pix_to_face [n, H, W, K] of a rank that packed only its own meshes -> global packed face ids:
    id - local_first[m] + global_first[m] per mesh m on occupied slots (-1 stays -1)."""
    import torch

    lf = torch.as_tensor(local_first, dtype=torch.int64, device=pix_to_face.device)
    gf = torch.as_tensor(global_first, dtype=torch.int64, device=pix_to_face.device)
    shift = (gf - lf).view(-1, *([1] * (pix_to_face.dim() - 1)))
    return torch.where(pix_to_face >= 0, pix_to_face + shift, pix_to_face)


def gather_fragments(local: dict, shards: list, rank: int, world: int, root: int = 0, face_ids=None):
    """Gather per-rank fragment blocks {name: tensor [n_r, ...]} into [N, ...] tensors on `root`, in global
    mesh order. Uses torch.distributed point-to-point sends (NCCL over NVLink on GPUs). ``face_ids`` =
    (local_first, global_first) of this rank's meshes: its 'pix_to_face' block is converted from rank-local to
    global packed face ids before it leaves the rank. Returns the gathered dict on root, None elsewhere."""
    import torch
    import torch.distributed as dist

    if face_ids is not None and "pix_to_face" in local and len(shards[rank]):
        local = dict(local)
        local["pix_to_face"] = globalize_face_ids(local["pix_to_face"], *face_ids)
    names = sorted(local)
    if rank != root:
        if not shards[rank]:
            return None
        reqs = [dist.isend(local[n].contiguous(), dst=root) for n in names]
        for r in reqs:
            r.wait()
        return None
    N = sum(len(s) for s in shards)
    out = {}
    for n in names:
        t = local[n]
        out[n] = torch.empty((N,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    for r in range(world):
        idx = shards[r]
        if not idx:
            continue
        for n in names:
            if r == root:
                buf = local[n]
            else:
                t = local[n]
                buf = torch.empty((len(idx),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
                dist.recv(buf, src=r)
            out[n][torch.as_tensor(idx, device=buf.device)] = buf
    return out
