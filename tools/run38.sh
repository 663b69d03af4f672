timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 160 --steps 3 --env "BLTC_FAR_DZS=0|BLTC_FAR_DZS=1|BLTC_FAR_DZS=0" > gpurun_out/sweep38.jsonl 2> gpurun_out/sweep38.err
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fast or mid_size" > gpurun_out/gpu_tests38.log 2>&1
