#!/bin/bash
# round-end style check: GPU suite, smoke, bench both arms (plain and torchrun N=1), launch list
TAG=${TAG:-final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_trun_$TAG.json 2> gpurun_out/bench_trun_$TAG.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/bench_trun_ref_$TAG.json 2> gpurun_out/bench_trun_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 > /dev/null 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
python - <<'PY'
import json
for f in ("bench", "bench_ref", "bench_trun", "bench_trun_ref"):
    try:
        d = json.load(open(f"gpurun_out/{f}_$TAG.json".replace("$TAG", __import__("os").environ.get("TAG", "final"))))
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("ms_per_step"), d.get("n_gpus"))
    except Exception as e:
        print(f, "ERR", e)
PY
