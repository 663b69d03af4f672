#!/usr/bin/env bash
# The measurement recipe behind profiles/r2_* (run on a B200 through gpurun):
#   bash tools/ref_suite/prepare.sh                      # here, once (reference tests)
#   /usr/local/graft/bin/gpurun --timeout 5400 -- 'bash tools/gpu_check.sh'
# Outputs land in gpurun_out/; summaries are copied to profiles/ by hand
# (tools/ncu_summary.py, tools/launch_summary.py).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
# headline (C4, STRICT) and the reference arm
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# every BASELINE config in STRICT, FAST and PARITY C4
for c in c1 c2 c3 c5 c4u; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 900 python bench.py --mode fast --steps 3 --no-cpu-baseline > gpurun_out/bench_fast_c4.json 2> gpurun_out/bench_fast_c4.err
timeout 900 python bench.py --mode parity --steps 2 --no-cpu-baseline --no-accuracy \
  > gpurun_out/bench_parity_c4.json 2> gpurun_out/bench_parity_c4.err
# STRICT certificate calibration: PARITY vs STRICT over all targets, Kc ratio
timeout 2400 python tools/strict_calibrate.py --configs c1,c2,c3,c4,c5 > gpurun_out/strict.jsonl 2> gpurun_out/strict.err
# fuzz: PARITY / STRICT / FAST against the oracle on edge cases; the STRICT
# certificate over random workloads (profiles/r2_*fuzz*.jsonl)
timeout 1700 python tools/parity_fuzz.py --runs 2000 > gpurun_out/parity_fuzz.jsonl 2> gpurun_out/parity_fuzz.err
timeout 1500 python tools/strict_fuzz.py --runs 120 > gpurun_out/strict_fuzz.jsonl 2> gpurun_out/strict_fuzz.err
timeout 2300 python tools/strict_fuzz.py --runs 150 --seed 7 --max-n 2000000 > gpurun_out/strict_fuzz_large.jsonl 2>&1
# accuracy cost of N_B; unsampled CPU steps anchoring the extrapolated baseline
timeout 900 python tools/nb_table.py --config c4 --batch-sizes 160,250,500,1000,2000 > gpurun_out/nb_c4.jsonl 2> gpurun_out/nb_c4.err
for c in c2 c3 c4; do
  timeout 900 python tools/cpu_full_step.py --config $c > gpurun_out/cpu_full_$c.json 2> gpurun_out/cpu_full_$c.err
done
# the reference's own test suite with its entry points bound to libbltc
BLTC_MODE=parity timeout 1500 bash tools/ref_suite/run.sh -q > gpurun_out/ref_suite_parity.log 2>&1
BLTC_MODE=strict timeout 1500 bash tools/ref_suite/run.sh -q > gpurun_out/ref_suite_strict.log 2>&1
# compute-sanitizer over every kernel family
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 2000 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
done
# N > 1 flow on one GPU (test hook, not a reported number)
BLTC_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --config c2 \
  --no-cpu-baseline > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err
# launch list (cold-cache, serialised: shares, not absolute times) and full captures
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_c4_strict.csv \
  python tools/one_step.py --config c4 --steps 2 --mode strict > gpurun_out/launches_c4.log 2>&1
# (reports summarised on the box and deleted: gpurun returns <= 64 MiB)
for k in k_far_packed k_near_packed k_moments_bw k_strict_recompute; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o /tmp/ncu_$k python tools/one_step.py --config c4 --steps 1 --mode strict > gpurun_out/ncu_$k.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$k.ncu-rep gpurun_out/ncu_${k}_c4.txt > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_far_packed -c 1 \
  -o /tmp/ncu_far_c3 python tools/one_step.py --config c3 --steps 1 --mode strict > gpurun_out/ncu_far_c3.log 2>&1
python tools/ncu_summary.py /tmp/ncu_far_c3.ncu-rep gpurun_out/ncu_far_yukawa_c3.txt > /dev/null 2>&1
