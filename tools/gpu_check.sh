#!/bin/bash
# Full round check on one B200: GPU tests, smoke, default bench (both arms), ncu launch list + full captures.
TAG=${TAG:-cur}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 > gpurun_out/ncu_bench.log 2>&1
if [ -n "$FULL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -s 1 -c 1 -o gpurun_out/prof_fine_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 > gpurun_out/ncu_fine_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_backward -s 1 -c 1 -o gpurun_out/prof_bwd_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 > gpurun_out/ncu_bwd_$TAG.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench_$TAG.json; cat gpurun_out/bench_ref_$TAG.json
