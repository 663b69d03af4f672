timeout 900 python bench.py > gpurun_out/b22_default.json 2> gpurun_out/b22_default.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --rank-path --no-cpu-baseline --no-accuracy > gpurun_out/b22_rank.json 2> gpurun_out/b22_rank.err
timeout 900 python bench.py --impl reference --steps 2 > gpurun_out/b22_ref.json 2> gpurun_out/b22_ref.err
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline > gpurun_out/b22_c3.json 2> gpurun_out/b22_c3.err
timeout 600 python bench.py --config c2 --steps 3 --no-cpu-baseline > gpurun_out/b22_c2.json 2> gpurun_out/b22_c2.err
