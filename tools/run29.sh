timeout 1500 python tools/sim_ranks.py --config c4 --ranks 1,2,4,8 > gpurun_out/sim_ranks_c4.jsonl 2> gpurun_out/sim_ranks_c4.err
