timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest3.txt
cat gpurun_out/pytest3.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err
python -c "import json; d=json.load(open('gpurun_out/bench3.json')); print(d['ms_per_step'], d['roofline']['per_kernel_ms_per_step'], d['clocks'])"
