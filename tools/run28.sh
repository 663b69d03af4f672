timeout 1200 python tools/sweep_c4.py --config c4 --leaf 1000,1500,2000,3000 --batch 140,160,180 --steps 2 > gpurun_out/sweep28.jsonl 2> gpurun_out/sweep28.err
