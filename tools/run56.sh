for N in 64 256; do
  rm -f paper_2003_01836_b200/_build/*.o
  BLTC_NVCC_DEFS="-DBLTC_EXP_N=$N" python -c "from paper_2003_01836_b200 import build_ext; build_ext.build()" > gpurun_out/build56_$N.log 2>&1
  timeout 900 python tools/sweep_c4.py --config c3 --leaf 2000 --batch 1000 --steps 3 --env "EXP_N=$N" >> gpurun_out/sweep56.jsonl 2>> gpurun_out/sweep56.err
  timeout 600 python -m pytest tests -q -m gpu -k "yukawa or Yukawa" > gpurun_out/gpu_tests56_$N.log 2>&1
done
