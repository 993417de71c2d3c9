"""bench.py's N > 1 code path on the GPU box (which has one GPU): two ranks launched by torch.distributed.run as the
driver launches them, sharing the GPU over gloo (DR_BENCH_SHARED_GPU=1; the NCCL gather needs one GPU per rank and
is covered at world size 1 by tests/test_gpu_shard.py). Checks the LPT plan, the sharded calls with global ranges,
max-over-ranks timing and that rank 0 alone prints the one JSON line; the timings are not scaling numbers."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_shared_gpu():
    env = dict(os.environ, DR_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", "C2", "--no-cpu-baseline", "--other-configs", "0", "--like-for-like", "0"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["workload"] == "C2" and d["e2e"]["value"] > 0
