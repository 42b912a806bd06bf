O=gpurun_out/split7; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:conv_tab_split --launch-skip 2 --launch-count 1 -o $O/split_rne python tools/conv_variants.py --config C5 --format e5m10 --variant 0 --reps 2 --f32 > $O/ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -f -k regex:conv_tab_kernel --launch-skip 2 --launch-count 1 -o $O/v4_rne python tools/conv_variants.py --config C5 --format e5m10 --variant 4 --reps 2 --f32 > $O/ncu4.log 2>&1
