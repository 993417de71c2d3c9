"""CPU suite: mesh sharding (LPT by face count, C-ABI plan), the gather's op list (dr_shard_gather_ops), and the
rank->root gather of REAL rasterizer output (the oracle, on CPU) over gloo with world_size 2."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2007_08501_b200 import scenes as S
from paper_2007_08501_b200.shard import COPY, RECV, SEND, ShardPlan, gather_ops, lpt_partition, shard_loads


def test_lpt_partition_balances_c4():
    counts = S.config_meshes("C4").num_faces_per_mesh()
    assert counts.sum() == 6581760
    for world in (1, 2, 4, 8):
        shards = lpt_partition(counts, world)
        assert sorted(i for s in shards for i in s) == list(range(len(counts)))
        loads = shard_loads(counts, shards)
        assert max(loads) <= counts.sum() / world + counts.max()
        if world > 1:
            assert max(loads) / (counts.sum() / world) < 1.05
    assert lpt_partition([5, 1], 4) == [[0], [1], [], []]
    with pytest.raises(ValueError):
        ShardPlan([1, 2], 0)


@pytest.mark.parametrize("world,root", [(1, 0), (2, 0), (3, 1), (8, 0)])
def test_gather_ops_match_and_cover(world, root):
    """Every root RECV is matched, in posting order, by the sender's SEND of the same buffer and size; every mesh
    reaches the root exactly once per buffer; pipelined subsets (local_index ranges) partition the full list."""
    counts = S.config_meshes("C2").num_faces_per_mesh()
    first = np.concatenate([[0], np.cumsum(counts)[:-1]])
    plan = ShardPlan(counts, world)
    slots, pb = 16 * 16 * 4, 4
    full = {r: gather_ops(plan, first, counts, slots, pb, True, r, root) for r in range(world)}
    root_ops = full[root]
    assert {o[0] for o in root_ops} <= {RECV, COPY}
    for r in range(world):
        if r != root:
            assert all(o[0] == SEND and o[1] == root for o in full[r])
            recvs = [o for o in root_ops if o[0] == RECV and o[1] == r]
            assert [(o[2], o[3], o[6]) for o in full[r]] == [(o[2], o[3], o[6]) for o in recvs]
    seen = {}
    for o in root_ops:
        seen.setdefault(o[2], []).append(o[3])
    for buf in ("pix_to_face", "zbuf", "bary", "dists", "grad_face_verts"):
        assert sorted(seen[buf]) == list(range(len(counts)))
    eb = {"pix_to_face": 8, "zbuf": pb, "bary": 3 * pb, "dists": pb}
    for o in root_ops:
        if o[2] in eb:
            assert o[5] == o[3] * slots * eb[o[2]] and o[6] == slots * eb[o[2]]
        else:
            assert o[4] == o[5] == first[o[3]] * 72 and o[6] == counts[o[3]] * 72
    nloc = max(int(plan.local_index.max()) + 1, 1)
    for r in range(world):
        parts = []
        for lo in range(0, nloc, 2):  # groups of two local meshes
            parts += gather_ops(plan, first, counts, slots, pb, True, r, root, lo, lo + 2)
        assert sorted(parts) == sorted(full[r])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


H, K, BLUR = 48, 4, 1e-4


def _scene():
    m, cam = S.config_meshes("C2"), S.bench_camera()
    fv = S.face_verts(m, cam)
    return fv, m.mesh_to_face_first_idx(), m.num_faces_per_mesh(), cam


def _worker(rank, world, port, result_q):
    import torch.distributed as dist

    from oracle.oracle import Oracle, make_settings
    from paper_2007_08501_b200.shard import gather_torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fv, first, num, cam = _scene()
    orc = Oracle()
    st = make_settings(H, H, K, BLUR, znear=cam.znear)
    plan = ShardPlan(num, world)
    mine = plan.meshes(rank)
    # this rank's meshes with their GLOBAL face ranges of the whole packed batch (the sharded call), real output
    p2f, zb, ba, di = orc.forward(fv, first[mine], num[mine], st)
    g = np.random.default_rng(9)
    S_ = len(num) * H * H * K
    dz, db, dd = g.standard_normal(S_), g.standard_normal(3 * S_), g.standard_normal(S_)
    per = H * H * K
    sl = np.concatenate([np.arange(m * per, (m + 1) * per) for m in mine]) if mine else np.zeros(0, np.int64)
    grad = orc.backward(fv, first[mine], num[mine], st, p2f, ba, dz[sl], db.reshape(-1, 3)[sl].reshape(-1), dd[sl])
    local = {"pix_to_face": torch.from_numpy(p2f), "zbuf": torch.from_numpy(zb), "bary": torch.from_numpy(ba),
             "dists": torch.from_numpy(di), "grad_face_verts": torch.from_numpy(grad)}
    glob = None
    N = len(num)
    if rank == 0:
        glob = {"pix_to_face": torch.full((N, H, H, K), -7, dtype=torch.int64),
                "zbuf": torch.zeros((N, H, H, K), dtype=torch.float64),
                "bary": torch.zeros((N, H, H, K, 3), dtype=torch.float64),
                "dists": torch.zeros((N, H, H, K), dtype=torch.float64),
                "grad_face_verts": torch.zeros_like(local["grad_face_verts"])}
    # pipelined as a caller would: one gather per pair of local meshes
    nloc = int(plan.local_index.max()) + 1
    for lo in range(0, nloc, 2):
        gather_torch(gather_ops(plan, first, num, per, 8, True, rank, 0, lo, lo + 2), local, glob)
    if rank == 0:
        want = orc.forward(fv, first, num, st)
        gw = orc.backward(fv, first, num, st, want[0], want[2], dz, db, dd)
        res = {"frag_equal": [bool(np.array_equal(glob[k].numpy(), w)) for k, w in
                              zip(("pix_to_face", "zbuf", "bary", "dists"), want)],
               "grad_max_err": float(np.abs(glob["grad_face_verts"].numpy() - gw).max()),
               "grad_scale": float(np.abs(gw).max()), "occupied": int((want[0] >= 0).sum())}
        result_q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def test_gather_real_fragments_gloo():
    """world_size 2 over gloo: each rank rasterizes ITS meshes (global face ranges) with the oracle, runs the
    backward, and gathers fragments + grad_face_verts rows to rank 0 in pipelined groups; rank 0's assembled batch
    equals the unsharded oracle forward bit for bit and the backward to the last bits."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(res["frag_equal"]), res
    assert res["occupied"] > 0
    assert res["grad_max_err"] <= 1e-12 * res["grad_scale"], res
