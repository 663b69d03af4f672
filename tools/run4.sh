timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
timeout 300 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 300 python bench.py --steps 3 --batch-size 1000 --no-cpu-baseline > gpurun_out/b_c4_nb1000.json 2> gpurun_out/b_c4_nb1000.err
