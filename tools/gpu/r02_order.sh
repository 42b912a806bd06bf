python bench.py --config C2 --steps 50 --no-cpu-baseline --no-sass > gpurun_out/o_c2.json 2>&1
python bench.py --steps 20 --no-cpu-baseline --no-sass > gpurun_out/o_c3.json 2>&1
python bench.py --config C4 --steps 10 --no-cpu-baseline --no-sass > gpurun_out/o_c4.json 2>&1
for n in 4 8; do python tools/conv_variants.py --config C3 --n $n --reps 10 2>&1 | tail -1; done > gpurun_out/o_small.txt
python bench.py --config C5 --sweep --steps 5 --no-cpu-baseline > gpurun_out/o_c5.json 2>&1
python bench.py --config MOBDW --steps 50 --no-cpu-baseline --no-sass > gpurun_out/o_mobdw.json 2>&1
python bench.py --kernel gates --steps 20 --no-cpu-baseline --no-sass > gpurun_out/o_c3g.json 2>&1
