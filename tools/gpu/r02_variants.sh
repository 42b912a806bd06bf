# conv schedule comparison on the C5 sweep layer (kernel-only timing, tools/conv_variants.py)
for fm in e4m8 e4m9 e4m10 e5m8 e5m9 e5m10 e6m8 e6m9 e6m10 e5m3 e5m7 e6m6; do
  for v in 0 4 9; do
    python tools/conv_variants.py --config C5 --format $fm --variant $v --reps 5 2>&1 | tail -1
  done
done > gpurun_out/variants_c5.txt
python -m pytest tests/test_gpu_parity.py -x -q -k "records or every_schedule or f32 or quantize" 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_c3.json 2>&1
python bench.py --config C4 --steps 10 --no-cpu-baseline > gpurun_out/b_c4.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sass > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sass > /dev/null 2>&1
