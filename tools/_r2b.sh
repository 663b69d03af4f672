set -x
timeout 900 python -m pytest tests/test_gpu_strict.py tests/test_gpu_parity.py tests/test_gpu_direct.py tests/test_gpu_stages.py tests/test_gpu_distributed.py -x -q > gpurun_out/r2b_tests.log 2>&1
tail -15 gpurun_out/r2b_tests.log
timeout 1200 python tools/strict_calibrate.py --configs c2,c3,c4 > gpurun_out/r2b_strict.jsonl 2> gpurun_out/r2b_strict.err
cat gpurun_out/r2b_strict.jsonl; tail -5 gpurun_out/r2b_strict.err
