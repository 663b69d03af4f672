timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests21.log 2>&1
timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 250 --steps 3 --env "BLTC_MOMENTS_OLD=0|BLTC_MOMENTS_OLD=1" > gpurun_out/sweep21.jsonl 2> gpurun_out/sweep21.err
