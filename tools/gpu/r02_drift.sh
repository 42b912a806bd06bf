# round-2d: is the L1-served wF = 10 kernel's L2 hit rate (39%) a tail effect or CTA drift?
# C5 e5m10 at 60 images (736 units: one co-resident wave of 740 slots) vs 64 (784 units)
O=gpurun_out/drift; mkdir -p $O
for n in 60 64; do for v in 4 0; do
  timeout 300 python tools/conv_variants.py --config C5 --format e5m10 --variant $v --n $n --reps 5 --f32 2>&1 | tail -1
done; done > $O/times.txt
for n in 60 64; do for v in 4 0; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:conv_tab --launch-skip 2 --launch-count 1 --csv --log-file $O/ncu_n${n}_v${v}.csv python tools/conv_variants.py --config C5 --format e5m10 --variant $v --n $n --reps 2 --f32 > /dev/null 2>&1
done; done
