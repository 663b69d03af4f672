timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests11.log 2>&1
timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 125,250,500,1000 --env "BLTC_PACK=1|BLTC_PACK=0" > gpurun_out/sweep11.jsonl 2> gpurun_out/sweep11.err
