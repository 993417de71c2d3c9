"""A/B of the host pipeline on C4: the native dr_host_pipeline (paper_2007_08501_b200.pipeline.HostPipeline) vs the
round-1 Python/torch-streams implementation (tools/pipeline_py_ab.py), alternating, same buffers, CUDA events."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench import config_settings  # noqa: E402
from paper_2007_08501_b200 import scenes as S  # noqa: E402
from paper_2007_08501_b200.pipeline import HostPipeline  # noqa: E402
import pipeline_py_ab  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
c = S.CONFIGS[cfg]
H = W = c["image"]
K = c["K"]
m, cam, rs = S.config_meshes(cfg), S.bench_camera(), config_settings(cfg)
fv = S.face_verts(m, cam)
first, num = m.mesh_to_face_first_idx(), m.num_faces_per_mesh()
N, F = len(num), len(fv)
dev = torch.device("cuda:0")
g = np.random.default_rng(1)
h_fv = torch.from_numpy(fv).pin_memory()
cot = tuple(torch.from_numpy(g.standard_normal(s).astype(np.float32)).pin_memory()
            for s in ((N, H, W, K), (N, H, W, K, 3), (N, H, W, K)))
out = (torch.empty((N, H, W, K), dtype=torch.int64).pin_memory(),
       torch.empty((N, H, W, K), dtype=torch.float32).pin_memory(),
       torch.empty((N, H, W, K, 3), dtype=torch.float32).pin_memory(),
       torch.empty((N, H, W, K), dtype=torch.float32).pin_memory())
grad = torch.empty((F, 3, 3), dtype=torch.float64).pin_memory()
res = {}
for name, mk in (("native", lambda: HostPipeline(first, num, rs, F, dev, n_groups=24)),
                 ("python", lambda: pipeline_py_ab.HostPipeline(first, num, rs, F, dev, n_groups=24))):
    pipe = mk()
    pipe.run(h_fv, out, cot, grad)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.run(h_fv, out, cot, grad)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[name] = ts
    del pipe
    torch.cuda.empty_cache()
print(json.dumps({k: {"median_ms": float(np.median(v)), "all": v} for k, v in res.items()}))
