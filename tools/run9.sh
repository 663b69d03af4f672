timeout 600 python -m pytest tests -x -q -m gpu -k "context_reuse or mid_size or deterministic" > gpurun_out/gpu_tests9.log 2>&1
timeout 900 python tools/sweep_c4.py --config c4 --leaf 1000,1500,2000,3000,4000 --batch 250,500,1000 > gpurun_out/sweep_c4.jsonl 2> gpurun_out/sweep_c4.err
