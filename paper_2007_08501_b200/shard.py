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


def gather_fragments(local: dict, shards: list, rank: int, world: int, root: int = 0):
    """Gather per-rank fragment blocks {name: tensor [n_r, ...]} into [N, ...] tensors on `root`, in global
    mesh order. Uses torch.distributed point-to-point sends (NCCL over NVLink on GPUs). Returns the gathered
    dict on root, None elsewhere."""
    import torch
    import torch.distributed as dist

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
