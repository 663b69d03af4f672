timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k ragged > gpurun_out/gpu_tests45.log 2>&1
