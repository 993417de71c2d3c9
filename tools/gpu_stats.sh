#!/bin/bash
# work counters of the fine stage (build the variant first: tools/build_variant.sh stats -DDR_STATS=1)
mkdir -p gpurun_out
DR_RASTER_LIB=build/variants/stats/libdr_raster_b200.so timeout 600 python tools/fine_stats.py C4 C5 C3 C2 2>&1 | tail -40
