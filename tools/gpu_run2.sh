timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -40 > gpurun_out/pytest2.txt
cat gpurun_out/pytest2.txt
