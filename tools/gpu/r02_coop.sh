# round-2d: warp-cooperative cp.async table gathers (variant 15) vs variant 4 / automatic, C5 L1-served formats
O=gpurun_out/coop; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "fractional_wave" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
for fm in e5m10 e6m10 e4m10 e6m9; do for n in 60 64; do for v in 4 15 0 4 15 0; do
  timeout 300 python tools/conv_variants.py --config C5 --format $fm --variant $v --n $n --reps 5 --f32 2>&1 | tail -1
done; done; done > $O/times.txt
for n in 60; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:conv_tab --launch-skip 2 --launch-count 1 --csv --log-file $O/ncu_n${n}_v15.csv python tools/conv_variants.py --config C5 --format e5m10 --variant 15 --n $n --reps 2 --f32 > /dev/null 2>&1
done
