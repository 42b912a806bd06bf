# round-2d: progress throttle (variant 14) for the L1-served wF = 10 kernel vs variants 4 / automatic; e6m9 routed to the fractional wave
O=gpurun_out/thr; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "fractional_wave or every_schedule or C5_whole or throttle" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
for fm in e5m10 e6m10 e4m10; do for n in 60 64; do for v in 4 14 0 4 14 0; do
  timeout 300 python tools/conv_variants.py --config C5 --format $fm --variant $v --n $n --reps 5 --f32 2>&1 | tail -1
done; done; done > $O/times.txt
for n in 60 64; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:conv_tab --launch-skip 2 --launch-count 1 --csv --log-file $O/ncu_n${n}_v14.csv python tools/conv_variants.py --config C5 --format e5m10 --variant 14 --n $n --reps 2 --f32 > /dev/null 2>&1
done
timeout 300 python tools/conv_variants.py --config C5 --format e6m9 --variant 0 --reps 5 --f32 2>&1 | tail -1 > $O/e6m9.txt
