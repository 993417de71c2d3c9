timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest6.txt
cat gpurun_out/pytest6.txt
./build/test_raster_cpp | tail -8
