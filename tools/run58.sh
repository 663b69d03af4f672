timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests58.log 2>&1
timeout 900 python bench.py > gpurun_out/b58_c4.json 2> gpurun_out/b58_c4.err
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline > gpurun_out/b58_c3.json 2> gpurun_out/b58_c3.err
