set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err
timeout 300 python bench.py --config c3 --steps 3 --no-cpu-baseline --no-accuracy > gpurun_out/b_c3.json 2> /dev/null
timeout 300 python bench.py --config c2 --steps 3 --no-cpu-baseline --no-accuracy > gpurun_out/b_c2.json 2> /dev/null
