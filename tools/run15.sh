./tools/fp64_peak2 > gpurun_out/fp64_peak2.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/b15_default.json 2> gpurun_out/b15_default.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches15_c4.csv python tools/one_step.py --config c4 --steps 2 > gpurun_out/launch15_c4.log 2>&1
