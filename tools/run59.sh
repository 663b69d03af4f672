timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 160 --steps 3 --env "BLTC_FAR_DY=0|BLTC_FAR_DY=1|BLTC_FAR_DY=0|BLTC_FAR_DY=1" > gpurun_out/sweep59.jsonl 2> gpurun_out/sweep59.err
BLTC_FAR_DY=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fast or mid_size" > gpurun_out/gpu_tests59.log 2>&1
