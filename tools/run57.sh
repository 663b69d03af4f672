set -e
for V in "-DBLTC_NEAR_UNROLL=2" "-DBLTC_NEAR_UNROLL=4" "-DBLTC_NEAR_UNROLL=8"; do
  rm -f paper_2003_01836_b200/_build/*.o
  BLTC_NVCC_DEFS="$V" python -c "from paper_2003_01836_b200 import build_ext; build_ext.build()"
  timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 160 --steps 3 --env "V=${V#-D}" >> gpurun_out/sweep57.jsonl 2>> gpurun_out/sweep57.err
done
for V in "-DBLTC_EXP_N=64" "-DBLTC_EXP_N=256"; do
  rm -f paper_2003_01836_b200/_build/*.o
  BLTC_NVCC_DEFS="$V" python -c "from paper_2003_01836_b200 import build_ext; build_ext.build()"
  timeout 900 python tools/sweep_c4.py --config c3 --leaf 2000 --batch 1000 --steps 3 --env "V=${V#-D}" >> gpurun_out/sweep57.jsonl 2>> gpurun_out/sweep57.err
  timeout 600 python -m pytest tests -q -m gpu -k "yukawa or Yukawa" > "gpurun_out/gpu_tests57$V.log" 2>&1 || true
done
