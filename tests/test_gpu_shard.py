"""Mesh-sharded execution on the GPU: LPT shards run as separate calls with their global face
ranges and assembled by the gather's op list == the unsharded call (fragments bit-exact, gradients to the
accumulation order); the NCCL executor (libdr_shard_b200.so) at world size 1 (the root's own device copies)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2007_08501_b200 import scenes as S
from tests._common import boundary, grad_close, raster_settings

pytestmark = pytest.mark.gpu


def _run(fv, first, num, rs, cuda, cot, grad=None):
    from paper_2007_08501_b200 import rasterize_meshes, rasterize_meshes_backward

    d = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=cuda)  # noqa: E731
    p2f, z, b, di = rasterize_meshes(d(fv), d(first), d(num), rs)
    g = rasterize_meshes_backward(d(fv), d(first), d(num), rs, p2f, b, *cot, out=grad)
    return {"pix_to_face": p2f, "zbuf": z, "bary": b, "dists": di, "grad_face_verts": g}


@pytest.mark.parametrize("cfg,world", [("C2", 2), ("C2", 3), ("C4", 3), ("C4", 8)])  # C4/3: > 8 range intervals
def test_sharded_equals_unsharded(cfg, world, cuda):
    from paper_2007_08501_b200.shard import ShardPlan, assemble_local

    c = S.CONFIGS[cfg]
    m, cam = S.config_meshes(cfg), S.bench_camera()
    fv, first, num = boundary(m, cam)
    H, K = c["image"], c["K"]
    rs = raster_settings(H, K, c["blur"], cam, persp_correct=bool(c.get("perspective_correct", False)),
                         cull=bool(c.get("cull_backfaces", False)))
    N, F = len(num), len(fv)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(4)
    cot = [torch.randn(s, generator=gen, device=cuda) for s in ((N, H, H, K), (N, H, H, K, 3), (N, H, H, K))]
    want = _run(fv, first, num, rs, cuda, cot)
    plan = ShardPlan(num, world)
    per_rank = []
    for r in range(world):
        mine = plan.meshes(r)
        assert mine
        # the rank's meshes with their GLOBAL ranges of the whole packed batch; its own grad_face_verts array
        grad = torch.zeros((F, 3, 3), dtype=torch.float64, device=cuda)
        per_rank.append(_run(fv, first[mine], num[mine], rs, cuda, [t[mine] for t in cot], grad))
    glob = {k: torch.empty_like(v) for k, v in want.items()}
    glob["grad_face_verts"].zero_()
    assemble_local(plan, per_rank, glob, first, num, H * H * K, 4, True)
    for k in ("pix_to_face", "zbuf", "bary", "dists"):
        assert torch.equal(glob[k], want[k]), f"{cfg} world {world}: {k} differs"
    grad_close(glob["grad_face_verts"].cpu().numpy(), want["grad_face_verts"].cpu().numpy(),
               f"{cfg} world {world} grad", rtol=1e-12, atol_scale=1e-14)


def test_nccl_gather_world1_copies(cuda):
    """The NCCL executor at world size 1: the root's meshes arrive by device copies into the global buffers
    (pipelined calls over local_index ranges)."""
    from paper_2007_08501_b200.shard import NcclGather, ShardPlan

    m, cam = S.config_meshes("C2"), S.bench_camera()
    fv, first, num = boundary(m, cam)
    rs = raster_settings(64, 4, 1e-4, cam)
    N, F = len(num), len(fv)
    cot = [torch.randn(s, device=cuda) for s in ((N, 64, 64, 4), (N, 64, 64, 4, 3), (N, 64, 64, 4))]
    local = _run(fv, first, num, rs, cuda, cot)
    plan = ShardPlan(num, 1)
    glob = {k: torch.zeros_like(v) for k, v in local.items()}
    g = NcclGather(0, 1)
    try:
        st = torch.cuda.current_stream()
        for lo in range(0, N, 3):
            g.gather(plan, first, num, 64 * 64 * 4, 4, True, local, glob, st, local_lo=lo, local_hi=lo + 3)
        torch.cuda.synchronize()
    finally:
        g.close()
    for k in local:
        assert torch.equal(glob[k], local[k]), k
