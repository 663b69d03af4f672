timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 160 --steps 3 --env "BLTC_FAR_UNROLL=3|BLTC_FAR_UNROLL=9|BLTC_FAR_UNROLL=3" > gpurun_out/sweep40.jsonl 2> gpurun_out/sweep40.err
