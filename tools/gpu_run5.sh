timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest5.txt
cat gpurun_out/pytest5.txt
bash tools/ab.sh M1 M2
