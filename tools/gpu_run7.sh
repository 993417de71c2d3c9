timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest7.txt
cat gpurun_out/pytest7.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -3 gpurun_out/bench7.err
python -c "import json; d=json.load(open('gpurun_out/bench7.json')); print(d['ms_per_step'], d['roofline']['per_kernel_ms_per_step'], d['e2e'])"
