timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests53.log 2>&1
timeout 900 python bench.py --mode parity --steps 1 --no-accuracy --no-cpu-baseline > gpurun_out/b53_parity.json 2> gpurun_out/b53_parity.err
