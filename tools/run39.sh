for G in 4 6 8; do
  rm -f paper_2003_01836_b200/_build/eval_packed.o
  BLTC_NVCC_DEFS="-DBLTC_GMAX=$G" python -c "from paper_2003_01836_b200 import build_ext; build_ext.build()" > gpurun_out/build_g$G.log 2>&1
  timeout 900 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 125,160,250 --steps 2 --env "BLTC_G=$G" >> gpurun_out/sweep39.jsonl 2>> gpurun_out/sweep39.err
done
