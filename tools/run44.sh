timeout 900 python bench.py > gpurun_out/b44_default.json 2> gpurun_out/b44_default.err
