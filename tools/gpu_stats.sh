#!/bin/bash
mkdir -p gpurun_out
for z in 0 1; do
  echo "== DR_ZSORT=$z"
  DR_ZSORT=$z DR_RASTER_LIB=build/variants/stats/libdr_raster_b200.so timeout 600 python tools/fine_stats.py C4 C5 C3 C2 2>&1 | tail -40
done
