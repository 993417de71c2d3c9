timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest4.txt
cat gpurun_out/pytest4.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -3 gpurun_out/bench4.err
python -c "import json; d=json.load(open('gpurun_out/bench4.json')); print(d['ms_per_step'], d['roofline']['per_kernel_ms_per_step'], d['clocks'])"
