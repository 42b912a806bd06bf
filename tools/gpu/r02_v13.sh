# round-2d: fractional wave at 4 CTAs / SM (variant 13) vs 5 (variant 12 = auto) vs variant 4, C5 wide formats
O=gpurun_out/v13; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fractional_wave or every_schedule" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
for fm in e6m10 e5m10 e4m10 e6m9; do for r in 0 1; do for v in 13 0 4 13 0 4; do
  timeout 300 python tools/conv_variants.py --config C5 --format $fm --variant $v --round $r --reps 5 --f32 2>&1 | tail -1
done; done; done > $O/r02_c5_split13.txt
