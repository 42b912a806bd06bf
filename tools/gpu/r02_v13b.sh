# round-2d: the fractional-wave L1-served schedule (12: 5 CTAs / SM, 13: 4) vs the automatic (tap-staged, variant 8) on C5 wF = 8, 9
O=gpurun_out/v13b; mkdir -p $O
for fm in e4m9 e5m9 e6m9 e4m8 e5m8 e6m8; do for r in 0 1; do for v in 0 12 13 0 12 13; do
  timeout 300 python tools/conv_variants.py --config C5 --format $fm --variant $v --round $r --reps 5 --f32 2>&1 | tail -1
done; done; done > $O/r02_c5_split13_wf89.txt
