./tools/fp64_latency > gpurun_out/fp64_latency.jsonl 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests25.log 2>&1
timeout 900 python tools/sweep_c4.py --config c3 --leaf 2000 --batch 1000 --steps 3 --env "BLTC_PACK=2|BLTC_PACK=1" > gpurun_out/sweep25_c3.jsonl 2> gpurun_out/sweep25_c3.err
timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 250 --steps 3 > gpurun_out/sweep25_c4.jsonl 2> gpurun_out/sweep25_c4.err
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline > gpurun_out/b25_c3.json 2> gpurun_out/b25_c3.err
