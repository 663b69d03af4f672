timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests13.log 2>&1
timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 125,250,500 > gpurun_out/sweep13.jsonl 2> gpurun_out/sweep13.err
