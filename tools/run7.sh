for nb in 500 700 1000 1500; do
timeout 300 python bench.py --steps 2 --batch-size $nb --no-cpu-baseline --no-accuracy > gpurun_out/b_c4_nb$nb.json 2> /dev/null
done
timeout 300 python bench.py --config c4u --steps 2 --no-cpu-baseline --no-accuracy > gpurun_out/b_c4u.json 2> /dev/null
timeout 300 python bench.py --config c4u --steps 2 --batch-size 1000 --no-cpu-baseline --no-accuracy > gpurun_out/b_c4u_nb1000.json 2> /dev/null
timeout 300 python bench.py --config c3 --steps 2 --no-cpu-baseline --no-accuracy > gpurun_out/b_c3.json 2> /dev/null
