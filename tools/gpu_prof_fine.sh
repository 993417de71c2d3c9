#!/bin/bash
# one full ncu capture of k_fine and k_backward on C4 (source-level) -> gpurun_out/prof_*.ncu-rep
mkdir -p gpurun_out
TAG=${TAG:-cur}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -s 1 -c 1 -o gpurun_out/prof_fine_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 > gpurun_out/ncu_fine_$TAG.log 2>&1
if [ -n "$BWD" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_backward -s 1 -c 1 -o gpurun_out/prof_bwd_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 > gpurun_out/ncu_bwd_$TAG.log 2>&1
fi
tail -2 gpurun_out/ncu_fine_$TAG.log
