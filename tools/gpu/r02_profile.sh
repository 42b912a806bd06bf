# round-2 profiling batch: bench lines + ncu --set full captures, summarised on the box
set -x
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_c3.json 2>&1
python bench.py --config MOBDW --steps 50 --no-cpu-baseline > gpurun_out/b_mobdw.json 2>&1
N="ncu --set full --clock-control none --import-source on"
cap() {  # name kernel-regex args...
  name=$1; k=$2; shift 2
  timeout 300 $N -k regex:$k --launch-skip 2 --launch-count 1 -o /tmp/$name python tools/ncu_target.py "$@" > gpurun_out/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep "$name: $*" > gpurun_out/$name.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/$name.src.csv 2>/dev/null
  gzip -c /tmp/$name.src.csv > gpurun_out/$name.src.csv.gz
}
cap mobdw_dw conv_dw --config MOBDW
cap mobdw_pack pack_f32 --config MOBDW
cap c5_e5m10 conv_tab --config C5 --format e5m10
cap c5_e6m9 conv_tab --config C5 --format e6m9
cap c5_e5m3 conv_tab --config C5 --format e5m3
cap c2 conv_tab --config C2
cap c3_quant quantize_acts --config C3
cap c3_conv conv_tab --config C3
cap c4_conv conv_tab --config C4
du -sh gpurun_out
