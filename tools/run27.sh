timeout 1200 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 125,160,200,250,320,400 --steps 2 > gpurun_out/sweep27.jsonl 2> gpurun_out/sweep27.err
timeout 1200 python tools/sweep_c4.py --config c4 --leaf 1000,4000,8000 --batch 250 --steps 2 >> gpurun_out/sweep27.jsonl 2>> gpurun_out/sweep27.err
