set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 300 python bench.py --config c2 --steps 3 --no-cpu-baseline > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 300 python bench.py --config c3 --steps 3 --no-cpu-baseline > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
timeout 600 python bench.py --config c4 --steps 3 --no-cpu-baseline > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 600 python bench.py --config c4 --steps 3 --batch-size 1000 --no-cpu-baseline > gpurun_out/b_c4_nb1000.json 2> gpurun_out/b_c4_nb1000.err
tail -3 gpurun_out/*.err
