for U in 2 4 8; do
  rm -f paper_2003_01836_b200/_build/eval_packed.o
  BLTC_NVCC_DEFS="-DBLTC_NEAR_UNROLL=$U" python -c "from paper_2003_01836_b200 import build_ext; build_ext.build()" > gpurun_out/build54_$U.log 2>&1
  timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 160 --steps 3 --env "NEAR_U=$U" >> gpurun_out/sweep54.jsonl 2>> gpurun_out/sweep54.err
done
