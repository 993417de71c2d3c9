for v in head2 pipe_split head2 pipe_split head2 pipe_split; do
  DR_RASTER_LIB=build/variants/$v/libdr_raster_b200.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --other-configs 0 --like-for-like 0 > gpurun_out/e2e_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$v.json')); print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],2))"
done
