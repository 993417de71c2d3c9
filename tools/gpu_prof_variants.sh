#!/bin/bash
# ncu --set full of k_fine (C4) for each variant named on the command line
mkdir -p gpurun_out
for v in "$@"; do
  DR_RASTER_LIB=build/variants/$v/libdr_raster_b200.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -s 1 -c 1 -o gpurun_out/prof_fine_$v python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 ${AB_ARGS} > gpurun_out/ncu_fine_$v.log 2>&1
  tail -1 gpurun_out/ncu_fine_$v.log
done
