#!/bin/bash
# ab.sh V1 V2 ... : bench each build/variants/V/libdr_raster_b200.so (kernel ms per step); AB_ARGS adds bench
# flags (e.g. "--config C5"); results in gpurun_out/ab_<V><tag>.json
tag=$(echo "${AB_ARGS}" | tr -c 'A-Za-z0-9' '_')
for v in "$@"; do
  DR_RASTER_LIB=build/variants/$v/libdr_raster_b200.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --other-configs 0 --like-for-like 0 ${AB_ARGS} > gpurun_out/ab_$v$tag.json 2> gpurun_out/ab_$v$tag.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_$v$tag.json')); print('$v', d['config']['workload'], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_$v$tag.err
done
