timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 250 --steps 3 --env "BLTC_PFORM=0|BLTC_PFORM=2|BLTC_PFORM=0" > gpurun_out/sweep16.jsonl 2> gpurun_out/sweep16.err
