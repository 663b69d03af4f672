timeout 1500 python bench.py --config c5 --steps 2 --no-cpu-baseline --accuracy-sample 1000 > gpurun_out/b24_c5.json 2> gpurun_out/b24_c5.err
timeout 600 python bench.py --config c2 --steps 3 --no-cpu-baseline > gpurun_out/b24_c2.json 2> gpurun_out/b24_c2.err
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline > gpurun_out/b24_c3.json 2> gpurun_out/b24_c3.err
