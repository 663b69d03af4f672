timeout 900 python -m pytest tests/test_gpu_multiprocess.py -x -q > gpurun_out/gpu_tests32.log 2>&1
