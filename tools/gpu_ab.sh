#!/bin/bash
# parity + kernel times on C4/C5/C3/C2 for the current build
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k division > gpurun_out/pytest_div.log 2>&1; tail -2 gpurun_out/pytest_div.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for cfg in ${CFGS:-C4 C5 C3 C2}; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 > gpurun_out/ab_$cfg.json 2> gpurun_out/ab_$cfg.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_$cfg.json')); print('$cfg', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_$cfg.err
done
