timeout 900 python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_distributed.py -x -q > gpurun_out/gpu_tests35.log 2>&1
