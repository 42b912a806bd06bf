# round-2d last verification of HEAD: every GPU test, smoke, default bench, C5 sweeps
O=gpurun_out/fin5; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "gpu tests exit $?" >> $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err
timeout 900 python bench.py --config C5 --sweep --steps 10 > $O/r02_bench_c5_sweep.json 2>&1
timeout 900 python bench.py --config C5 --sweep --steps 10 --round rtz > $O/r02_bench_c5_sweep_rtz.json 2>&1
