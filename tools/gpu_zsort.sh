#!/bin/bash
# depth-ordered fine stage: parity + A/B (DR_ZSORT=0 vs default)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for z in 0 1; do
  for cfg in C4 C5 C3 C2; do
    DR_ZSORT=$z timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_z${z}_$cfg.json 2> gpurun_out/ab_z${z}_$cfg.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_z${z}_$cfg.json')); print('z=$z $cfg', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_z${z}_$cfg.err
  done
done
