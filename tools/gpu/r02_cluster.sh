python -m pytest tests/test_gpu_parity.py -q -x -k "every_schedule" 2>&1 | tail -2
for fm in e4m8 e5m8 e6m8 e4m9 e5m9 e6m9 e4m10 e5m10 e6m10 e5m7; do for v in 0 12; do python tools/conv_variants.py --config C5 --format $fm --variant $v --reps 5 2>&1 | tail -1; done; done > gpurun_out/cluster_c5.txt
