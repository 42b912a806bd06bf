# schedules at a rank's share of C3 / C4 / C5 under the strong split (N = 2, 4, 8)
for n in 4 8 16; do for v in 0 4 5 6 7; do python tools/conv_variants.py --config C3 --n $n --variant $v --reps 10 2>&1 | tail -1; done; done > gpurun_out/small_c3.txt
for n in 32 64 128; do for v in 0 5 7; do python tools/conv_variants.py --config C4 --n $n --variant $v --reps 5 2>&1 | tail -1; done; done > gpurun_out/small_c4.txt
for n in 8 16 32; do for v in 0 5 7; do python tools/conv_variants.py --config C5 --format e5m3 --n $n --variant $v --reps 10 2>&1 | tail -1; done; done > gpurun_out/small_c5.txt
