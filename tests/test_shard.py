"""CPU suite: mesh sharding (LPT by face count) and the rank->root fragment gather over gloo, world_size 2."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2007_08501_b200 import scenes as S
from paper_2007_08501_b200.shard import gather_fragments, lpt_partition, shard_loads


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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shards, result_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # each rank fabricates the fragment blocks of its meshes: value = global mesh id
    idx = shards[rank]
    # rank-local packing: this rank's meshes own faces [local_first[m], ...) of ITS face_verts; every occupied
    # slot holds the mesh's first local face id, one slot per pixel is empty
    counts = np.array([100, 5, 70, 30, 1])
    gfirst = np.concatenate([[0], np.cumsum(counts)[:-1]])
    lcounts = counts[idx]
    lfirst = np.concatenate([[0], np.cumsum(lcounts)[:-1]]) if len(idx) else np.zeros(0, np.int64)
    p2f = torch.tensor(lfirst, dtype=torch.int64).view(-1, 1, 1, 1).expand(-1, 4, 4, 2).contiguous()
    p2f[:, :, :, 1] = -1
    loc = {"pix_to_face": p2f,
           "zbuf": torch.tensor(idx, dtype=torch.float32).view(-1, 1, 1, 1).expand(-1, 4, 4, 2).contiguous()}
    out = gather_fragments(loc, shards, rank, world, root=0, face_ids=(lfirst, gfirst[idx]))
    if rank == 0:
        result_q.put({k: v.numpy() for k, v in out.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gather_fragments_gloo(world):
    counts = [100, 5, 70, 30, 1]
    shards = lpt_partition(counts, world)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shards, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = len(counts)
    gfirst = np.concatenate([[0], np.cumsum(counts)[:-1]])
    assert np.array_equal(res["pix_to_face"][:, 0, 0, 0], gfirst)  # global packed ids on the root
    assert np.all(res["pix_to_face"][:, :, :, 1] == -1)
    assert np.array_equal(res["zbuf"][:, 3, 3, 1], np.arange(n, dtype=np.float32))
