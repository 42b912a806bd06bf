# quantiser A/B: direct scalar kernel (current libhobf.so) vs the bitsliced one (tools/ab/libhobf_old.so)
python -m pytest tests/test_gpu_parity.py -x -q -k "records or quantis or wide_rows" > gpurun_out/qt_tests.log 2>&1; tail -1 gpurun_out/qt_tests.log
python tools/edge_bench.py --configs C3,C4,C5,MOB --flush read > gpurun_out/qt_new_r.txt 2>&1
N="ncu --set full --clock-control none --import-source on -f"
cap() {
  name=$1; k=$2; shift 2
  timeout 300 $N -k regex:$k --launch-skip 2 --launch-count 1 -o /tmp/$name python tools/ncu_target.py "$@" > gpurun_out/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep "$name: $*" > gpurun_out/$name.txt 2>&1
}
cap qd_c3 quantize_acts_direct --config C3
cp tools/ab/libhobf_old.so paper_2007_06563_b200/libhobf.so
python tools/edge_bench.py --configs C3,C4,C5,MOB --flush read > gpurun_out/qt_old_r.txt 2>&1
cat gpurun_out/qt_new_r.txt gpurun_out/qt_old_r.txt | grep quantize_act
