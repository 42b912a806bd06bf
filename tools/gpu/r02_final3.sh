# round-2c final: every GPU test, smoke, bench lines (C3, C5 sweeps), variant-12 timings
O=gpurun_out/fin3; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "gpu tests exit $?" >> $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err
for fm in e5m10 e4m10 e6m10 e6m9; do for r in 0 1; do for v in 4 0 4 0; do
  timeout 300 python tools/conv_variants.py --config C5 --format $fm --variant $v --round $r --reps 5 --f32 2>&1 | tail -1
done; done; done > $O/r02_c5_split.txt
timeout 900 python bench.py --config C5 --sweep --steps 10 > $O/r02_bench_c5_sweep.json 2>&1
timeout 900 python bench.py --config C5 --sweep --steps 10 --round rtz > $O/r02_bench_c5_sweep_rtz.json 2>&1
