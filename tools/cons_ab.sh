#!/bin/bash
# fused silhouette + softmax consumer kernel times (tools/bench_consumers.py) for build variants: cons_ab.sh V1 V2 ...
for v in "$@"; do
  DR_RASTER_LIB=build/variants/$v/libdr_raster_b200.so python tools/bench_consumers.py --config ${CFG:-C4} --steps 5 > gpurun_out/cons_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/cons_$v.json'))
print('$v', '${CFG:-C4}', 'sil', round(d['fused_ms'],3), {k: round(x,3) for k,x in d['fused_kernels_ms'].items() if k in ('k_fine','k_silhouette_backward')}, 'soft', round(d['softmax_fused_ms'],3), {k: round(x,3) for k,x in d['softmax_fused_kernels_ms'].items() if k in ('k_fine','k_softmax_backward')})"
done
