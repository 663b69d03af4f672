timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests31.log 2>&1
timeout 900 python bench.py > gpurun_out/b31_default.json 2> gpurun_out/b31_default.err
