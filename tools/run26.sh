timeout 900 python tools/sweep_c4.py --config c3 --leaf 2000 --batch 1000 --steps 3 --env "BLTC_PACK=2|BLTC_PACK=1" > gpurun_out/sweep26_c3.jsonl 2> gpurun_out/sweep26_c3.err
timeout 600 python -m pytest tests -x -q -m gpu -k "yukawa or Yukawa or dist" > gpurun_out/gpu_tests26.log 2>&1
