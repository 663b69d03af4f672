timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 250 --steps 3 --env "BLTC_FAR_MINB=2|BLTC_FAR_MINB=1" > gpurun_out/sweep17.jsonl 2> gpurun_out/sweep17.err
