timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 160 --steps 3 --env "BLTC_NEAR_NSM=0|BLTC_NEAR_NSM=1|BLTC_NEAR_NSM=0" > gpurun_out/sweep41.jsonl 2> gpurun_out/sweep41.err
BLTC_NEAR_NSM=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -x -q -k "fast or mid_size or simulated" > gpurun_out/gpu_tests41.log 2>&1
