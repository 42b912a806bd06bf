N="ncu --set full --clock-control none --import-source on -f"
cap() {
  name=$1; k=$2; shift 2
  timeout 300 $N -k regex:$k --launch-skip 2 --launch-count 1 -o /tmp/$name python tools/ncu_target.py "$@" > gpurun_out/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep "$name: $*" > gpurun_out/$name.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
}
cap qd_c3 quantize_acts_direct --config C3
cap qd_c4 quantize_acts_direct --config C4
