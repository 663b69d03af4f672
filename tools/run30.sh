timeout 900 python -m pytest tests -x -q -m gpu -k "dist or cli" > gpurun_out/gpu_tests30.log 2>&1
timeout 1500 python tools/sim_ranks.py --config c4 --ranks 8 > gpurun_out/sim_ranks30.jsonl 2> gpurun_out/sim_ranks30.err
