timeout 900 python tools/sweep_c4.py --config c3 --leaf 2000 --batch 2000,1000,500 --steps 3 --env "BLTC_PACK=2|BLTC_PACK=1|BLTC_PACK=0" > gpurun_out/sweep23_c3.jsonl 2> gpurun_out/sweep23_c3.err
timeout 900 python tools/sweep_c4.py --config c2 --leaf 2000 --batch 2000,1000,500 --steps 3 --env "BLTC_PACK=2|BLTC_PACK=1|BLTC_PACK=0" > gpurun_out/sweep23_c2.jsonl 2> gpurun_out/sweep23_c2.err
timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 250 --steps 2 > gpurun_out/sweep23_c4.jsonl 2> gpurun_out/sweep23_c4.err
