# round-2d final: every GPU test, smoke, bench lines (C3, C5 sweeps) after the 4-CTA fractional wave (variant 13)
O=gpurun_out/fin4; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "gpu tests exit $?" >> $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err
timeout 900 python bench.py --config C5 --sweep --steps 10 > $O/r02_bench_c5_sweep.json 2>&1
timeout 900 python bench.py --config C5 --sweep --steps 10 --round rtz > $O/r02_bench_c5_sweep_rtz.json 2>&1
timeout 900 python bench.py --config C5 --sweep --steps 10 --extended 1 > $O/r02_bench_c5_sweep_extended.json 2>&1
timeout 600 python bench.py --config MOBDW --steps 50 --no-cpu-baseline > $O/r02_bench_mobdw.json 2>&1
timeout 600 python bench.py --config C4 --steps 50 --no-cpu-baseline > $O/r02_bench_c4.json 2>&1
# ncu --set full of the 4-CTA fractional wave (C5 e6m10, automatic schedule), after its command exited 0 above
timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:conv_tab_split --launch-skip 2 --launch-count 1 -o /tmp/split13_e6m10 python tools/conv_variants.py --config C5 --format e6m10 --variant 0 --reps 2 --f32 > $O/ncu.log 2>&1
python tools/ncu_summary.py /tmp/split13_e6m10.ncu-rep "r02_ncu_c5_e6m10_split13: tools/conv_variants.py --config C5 --format e6m10 --variant 0 --f32 (automatic: fractional wave at 4 CTAs / SM)" > $O/r02_ncu_c5_e6m10_split13.txt 2>&1
