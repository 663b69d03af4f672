timeout 900 python bench.py --mode parity --steps 1 --no-accuracy --no-cpu-baseline > gpurun_out/b46_parity.json 2> gpurun_out/b46_parity.err
timeout 900 python bench.py --config c2 --mode parity --steps 1 --no-accuracy --no-cpu-baseline > gpurun_out/b46_parity_c2.json 2> gpurun_out/b46_parity_c2.err
