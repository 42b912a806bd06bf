for fm in e4m10 e5m10 e6m10; do for r in 0 1; do python tools/conv_variants.py --config C5 --format $fm --variant 4 --round $r --reps 5 2>&1 | tail -1; done; done > gpurun_out/c5_v4.txt
python -m pytest tests/test_gpu_parity_full.py -x -q -k "C5" 2>&1 | tail -2
python bench.py --config C5 --sweep --steps 10 > gpurun_out/r02_bench_c5_sweep.json 2>&1
python bench.py --config C5 --sweep --steps 10 --round rtz > gpurun_out/r02_bench_c5_sweep_rtz.json 2>&1
