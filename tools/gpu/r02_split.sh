O=gpurun_out/split8; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fractional_wave and 5-10" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
for fm in e5m10; do for r in 0 1; do for v in 4 0 4 0; do
  timeout 300 python tools/conv_variants.py --config C5 --format $fm --variant $v --round $r --reps 5 --f32 2>&1 | tail -1
done; done; done > $O/c5_variants.txt
