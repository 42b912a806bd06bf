for fm in e5m10 e4m10 e6m10 e6m9; do for v in 0 12; do python tools/conv_variants.py --config C5 --format $fm --variant $v --reps 5; done; done > gpurun_out/v12.txt 2>&1
cat gpurun_out/v12.txt
