timeout 600 python -m pytest tests/test_gpu_generate.py -x -q > gpurun_out/gpu_tests37.log 2>&1
timeout 600 python bench.py --config c2 --steps 2 --no-cpu-baseline > gpurun_out/b37_c2.json 2> gpurun_out/b37_c2.err
