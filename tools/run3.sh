timeout 600 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err
timeout 600 python bench.py --impl reference > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/one_step.py --config c4 --steps 2 > gpurun_out/launch_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_far_fast -s 1 -c 1 -o gpurun_out/prof_far_c4 python tools/one_step.py --config c4 --steps 2 > gpurun_out/prof_far_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_near_fast -s 1 -c 1 -o gpurun_out/prof_near_c4 python tools/one_step.py --config c4 --steps 2 > gpurun_out/prof_near_c4.log 2>&1
