export PYTHONUNBUFFERED=1
nproc > gpurun_out/nproc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1v4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -s 1 -c 1 -o gpurun_out/prof_fine_v4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fine_v4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_backward -s 1 -c 1 -o gpurun_out/prof_bwd_v4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bwd_v4.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_v4.json 2> gpurun_out/bench_ref_v4.err
cat gpurun_out/bench_v4.json gpurun_out/bench_ref_v4.json; tail -3 gpurun_out/bench_v4.err
