#!/usr/bin/env bash
# The measurement recipe behind profiles/ (run on a B200 through gpurun):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/gpu_check.sh'
# Outputs land in gpurun_out/; summaries are copied to profiles/ by hand
# (tools/ncu_summary.py, tools/launch_summary.py).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 900 python bench.py --mode parity --steps 2 --no-cpu-baseline --no-accuracy \
  > gpurun_out/bench_parity_c4.json 2> gpurun_out/bench_parity_c4.err
# the paper's Fig. 3 theta x degree sweep through the harness
timeout 900 python -m paper_2003_01836_b200 sweep --n-particles 1000000 --thetas 0.5,0.7,0.9 \
  --degrees 1,2,3,4,5,6,7,8,9,10,11,12 --batch-size 160 --verify 4000 --format csv \
  --output gpurun_out/sweep_fig3_1m.csv > gpurun_out/sweep_fig3.log 2>&1
# N > 1 flow on one GPU (test hook, not a reported number)
BLTC_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --config c2 \
  --no-cpu-baseline > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err
# launch list (cold-cache, serialised: shares, not absolute times)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
  python tools/one_step.py --config c4 --steps 2 > gpurun_out/launches_c4.log 2>&1
# full captures of the two interaction kernels and the upward pass
for k in k_far_packed k_near_packed k_moments_warp; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o gpurun_out/ncu_$k python tools/one_step.py --config c4 --steps 1 > gpurun_out/ncu_$k.log 2>&1
done
# projected multi-GPU step from simulated ranks
timeout 1500 python tools/sim_ranks.py --config c4 --ranks 1,2,4,8 > gpurun_out/sim_ranks_c4.jsonl 2> gpurun_out/sim_ranks_c4.err
