# round-2 re-entry: verify HEAD on one B200 (gpu tests, smoke, default bench)
O=gpurun_out/ver; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "gpu tests exit $?" >> $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config MOBDW --steps 50 --no-cpu-baseline > $O/bench_mobdw.json 2>&1
