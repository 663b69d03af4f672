timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests20.log 2>&1
timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 250 --steps 3 > gpurun_out/sweep20.jsonl 2> gpurun_out/sweep20.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches20_c4.csv python tools/one_step.py --config c4 --steps 2 --batch-size 250 > gpurun_out/launch20_c4.log 2>&1
