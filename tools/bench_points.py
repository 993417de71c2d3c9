"""Point rasterizer throughput on one B200 vs the reference CPU implementation.

  python tools/bench_points.py [--clouds 32] [--points 100000] [--image 256] [--K 8] [--radius 0.01]

GPU: rasterize_points (fp32 payload) + rasterize_points_backward, inputs resident, CUDA events.
CPU: the reference's own dr::rasterize_points (oracle/_ref, all host threads) on a sample of the clouds.
Metric: Mpoints·px/s = sum_b P_b * H * W / t / 1e6 (the naive pair count, like the mesh path's metric).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2007_08501_b200 import (PointRasterSettings, rasterize_points, rasterize_points_backward,  # noqa: E402
                                   scenes as S)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clouds", type=int, default=32)
    ap.add_argument("--points", type=int, default=100000)
    ap.add_argument("--image", type=int, default=256)
    ap.add_argument("--K", type=int, default=8)
    ap.add_argument("--radius", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    clouds = [rng.standard_normal((a.points, 3)) * 0.5 for _ in range(a.clouds)]
    pts = np.concatenate(clouds)
    num = np.full(a.clouds, a.points, np.int64)
    first = np.arange(a.clouds, dtype=np.int64) * a.points
    cam = S.bench_camera()
    ndc = S.points_ndc(pts, cam)
    dev = torch.device("cuda:0")
    x = torch.as_tensor(ndc, device=dev)
    rs = PointRasterSettings(image_size=a.image, points_per_pixel=a.K, radius=a.radius, bin_size=16)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    shp = (a.clouds, a.image, a.image, a.K)
    gz, gd = torch.randn(shp, generator=g, device=dev), torch.randn(shp, generator=g, device=dev)

    def step():
        idx, zb, d2 = rasterize_points(x, first, num, rs)
        return rasterize_points_backward(x, first, num, rs, idx, gz, gd)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    pairs = float(len(pts)) * a.image * a.image
    out = {"metric": "rasterize_points fwd+bwd Mpoints·px/s", "value": pairs / (ms * 1e-3) / 1e6, "ms_per_step": ms,
           "config": {"clouds": a.clouds, "points_per_cloud": a.points, "image": a.image, "K": a.K,
                      "radius": a.radius}}
    try:  # the reference's own CPU implementation on a sample (forward only: it has no point backward)
        from oracle.oracle import RefLib

        ref = RefLib()
        ns = max(1, a.clouds // 8)
        t0 = time.perf_counter()
        ref.rasterize_points(np.concatenate(clouds[:ns]), num[:ns], cam.packed(), a.image, a.image, a.K, a.radius)
        t = time.perf_counter() - t0
        out["cpu_reference_fwd"] = {"value": ns * a.points * a.image * a.image / t / 1e6, "clouds": ns, "s": t,
                                    "threads": ref.num_threads()}
    except Exception as e:  # noqa: BLE001
        out["cpu_reference_fwd"] = {"unavailable": str(e)}
    from paper_2007_08501_b200 import KernelTimer

    torch.cuda.synchronize()
    with KernelTimer() as kt:
        for _ in range(5):
            step()
        torch.cuda.synchronize()
    per = {}
    for k, t in kt.records:
        per[k] = round(per.get(k, 0.0) + t / 5, 4)
    out["kernels_ms"] = per
    print(json.dumps(out))


if __name__ == "__main__":
    main()
