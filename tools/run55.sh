timeout 1500 python bench.py --config paper64m --steps 2 --no-cpu-baseline --accuracy-sample 1000 > gpurun_out/b55_paper64m.json 2> gpurun_out/b55_paper64m.err
timeout 1500 python tools/sweep_c4.py --config paper64m --leaf 2000,4000 --batch 1000,4000 --steps 1 > gpurun_out/sweep55.jsonl 2> gpurun_out/sweep55.err
timeout 1500 python bench.py --config paper64m_y --steps 2 --no-cpu-baseline --accuracy-sample 1000 > gpurun_out/b55_paper64m_y.json 2> gpurun_out/b55_paper64m_y.err
