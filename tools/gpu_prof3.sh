timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -s 1 -c 1 -o gpurun_out/prof_fine_v3 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fine_v3.log 2>&1
tail -2 gpurun_out/ncu_fine_v3.log
