# after the GPU-proved sweeps of the wider table MACs: GPU tests, C5 sweep lines, the default bench
O=gpurun_out/fin3; mkdir -p $O
(time python -m pytest tests -m gpu -x -q) > $O/gputest.log 2>&1; tail -3 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; cat $O/smoke.log
B="python bench.py"
$B --config C5 --sweep --steps 10 > $O/r02_bench_c5_sweep.json 2>&1
$B --config C5 --sweep --steps 10 --round rtz > $O/r02_bench_c5_sweep_rtz.json 2>&1
$B --config C5 --sweep --steps 5 --extended 1 > $O/r02_bench_c5_sweep_extended.json 2>&1
$B > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err
