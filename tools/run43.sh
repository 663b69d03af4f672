BLTC_TRACE_MASK=1 timeout 600 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 160 --steps 1 > gpurun_out/sweep43a.jsonl 2> gpurun_out/sweep43a.err
rm -f paper_2003_01836_b200/_build/eval_packed.o
BLTC_NVCC_DEFS="-DBLTC_DEBUG_NOMASK" python -c "from paper_2003_01836_b200 import build_ext; build_ext.build()" > gpurun_out/build43.log 2>&1
timeout 600 python tools/sweep_c4.py --config c4 --leaf 2000 --batch 160 --steps 3 > gpurun_out/sweep43b.jsonl 2> gpurun_out/sweep43b.err
