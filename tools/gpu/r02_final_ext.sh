O=gpurun_out/fin4; mkdir -p $O
(time python -m pytest tests -m gpu -x -q) > $O/gputest.log 2>&1; tail -3 $O/gputest.log
B="python bench.py --no-cpu-baseline"
$B --extended 1 > $O/r02_bench_c3_extended.json 2>&1
$B --config C5 --sweep --steps 5 --extended 1 > $O/r02_bench_c5_sweep_extended.json 2>&1
