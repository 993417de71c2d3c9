"""fit_silhouette (pipeline.cpp:100-205) wall time: the B200 path vs the reference library on the host.

  python tools/bench_fit.py [--iterations 400] [--ref-threads N]   -> one JSON line
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2007_08501_b200.fit import FitConfig, fit_silhouette  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterations", type=int, default=400)
    ap.add_argument("--ref-threads", type=int, default=os.cpu_count())
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    cfg = FitConfig(iterations=a.iterations)  # the reference defaults: sphere:2 target, 2 views, 64x64, K=24
    fit_silhouette(FitConfig(iterations=3), "cuda")  # warm-up (library load, allocator)
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = fit_silhouette(cfg, "cuda")
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t
    out = {"fit": "defaults (pipeline.hpp:56-78)", "iterations": cfg.iterations, "gpu_s": gpu_s,
           "gpu_ms_per_iter": gpu_s / cfg.iterations * 1e3, "gpu_final_loss": res.final_silhouette_loss}
    if not a.no_ref:
        from oracle.oracle import RefLib

        R = RefLib()
        R.set_num_threads(a.ref_threads)
        t = time.perf_counter()
        _, final, _ = R.fit_silhouette(cfg)
        ref_s = time.perf_counter() - t
        out.update({"ref_s": ref_s, "ref_threads": a.ref_threads, "ref_final_loss": final,
                    "speedup": ref_s / gpu_s})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
