for n in 4 8 16 32; do for v in 5 10 11 12 4; do python tools/conv_variants.py --config C3 --n $n --variant $v --reps 10 2>&1 | tail -1; done; done > gpurun_out/shape_c3.txt
for n in 8 16 32 64; do for v in 5 10 11 12; do python tools/conv_variants.py --config C5 --format e5m3 --n $n --variant $v --reps 10 2>&1 | tail -1; done; done > gpurun_out/shape_c5.txt
for n in 32 64; do for v in 10 11 12; do python tools/conv_variants.py --config C4 --n $n --variant $v --reps 5 2>&1 | tail -1; done; done > gpurun_out/shape_c4.txt
for n in 16 32 64 128; do for v in 5 10 11 12; do python tools/conv_variants.py --config MOB --n $n --variant $v --reps 5 2>&1 | tail -1; done; done > gpurun_out/shape_mob.txt
