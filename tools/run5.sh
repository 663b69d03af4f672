timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --rank-path --steps 3 --no-cpu-baseline > gpurun_out/b_rank1.json 2> gpurun_out/b_rank1.err
