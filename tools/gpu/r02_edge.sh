# edge kernels (quantize / pack) after the pipelined bitsliced rewrite
python -m pytest tests/test_gpu_parity.py -x -q -k "records or f32 or quantize or pack or dw or C1_full" 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_c3.json 2>&1
python bench.py --config MOBDW --steps 50 --no-cpu-baseline > gpurun_out/b_mobdw.json 2>&1
python bench.py --config C4 --steps 10 --no-cpu-baseline > gpurun_out/b_c4.json 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv"
ncu $M --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sass > /dev/null 2>&1
ncu $M --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sass > /dev/null 2>&1
ncu $M --log-file gpurun_out/launches_mobdw.csv python bench.py --config MOBDW --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sass > /dev/null 2>&1
