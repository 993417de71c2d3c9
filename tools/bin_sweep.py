"""K2 time vs bin size on a bench config (bin_size is a performance knob: results are identical for any value).

  python tools/bin_sweep.py [--config C4] [--bins 8,16,32,64]
"""
import argparse
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import config_settings  # noqa: E402
from paper_2007_08501_b200 import KernelTimer, rasterize_meshes, rasterize_meshes_backward, scenes as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--bins", default="8,16,32,64")
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    m, cam = S.config_meshes(a.config), S.bench_camera()
    rs0 = config_settings(a.config)
    fv = torch.as_tensor(S.face_verts(m, cam), device=dev)
    first = torch.as_tensor(m.mesh_to_face_first_idx(), device=dev)
    num = torch.as_tensor(m.num_faces_per_mesh(), device=dev)
    H, W = rs0.hw
    K = rs0.faces_per_pixel
    N = len(num)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    dz = torch.randn((N, H, W, K), generator=g, device=dev)
    db = torch.randn((N, H, W, K, 3), generator=g, device=dev)
    dd = torch.randn((N, H, W, K), generator=g, device=dev)
    ref = None
    out = {}
    for b in [int(x) for x in a.bins.split(",")]:
        rs = dataclasses.replace(rs0, bin_size=b)
        p2f = rasterize_meshes(fv, first, num, rs)[0]
        if ref is None:
            ref = p2f
        same = bool(torch.equal(p2f, ref))
        del p2f
        torch.cuda.synchronize()
        with KernelTimer() as kt:
            for _ in range(a.steps):
                p2f, zb, bary, di = rasterize_meshes(fv, first, num, rs)
                rasterize_meshes_backward(fv, first, num, rs, p2f, bary, dz, db, dd)
            torch.cuda.synchronize()
        per = {}
        for k, ms in kt.records:
            per[k] = round(per.get(k, 0.0) + ms / a.steps, 3)
        out[b] = {"identical": same, "ms": round(sum(per.values()), 3), "kernels": per}
        del p2f, zb, bary, di
        torch.cuda.empty_cache()
    print(json.dumps({"config": a.config, "bins": out}))


if __name__ == "__main__":
    main()
