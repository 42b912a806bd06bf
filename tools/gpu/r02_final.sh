# round-2 final refresh (one B200): bench lines, strong-split correctness runs,
# launch lists and ncu --set full captures of the kernels that changed.
O=gpurun_out/fin2; mkdir -p $O
B="python bench.py"
$B > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err
$B --impl reference > $O/r02_bench_c3_reference_arm.json 2>&1
$B --round rtz --no-cpu-baseline > $O/r02_bench_c3_rtz.json 2>&1
$B --extended 1 --no-cpu-baseline > $O/r02_bench_c3_extended.json 2>&1
$B --kernel gates --no-cpu-baseline --steps 50 > $O/r02_bench_c3_gates.json 2>&1
$B --out planes --no-cpu-baseline > $O/r02_bench_c3_planes.json 2>&1
$B --relu 1 --no-cpu-baseline > $O/r02_bench_c3_relu.json 2>&1
for c in C1 C2 MOB MOBDW; do $B --config $c --steps 50 --no-cpu-baseline > $O/r02_bench_$(echo $c | tr A-Z a-z).json 2>&1; done
$B --config C2 --steps 50 --kernel gates --no-cpu-baseline > $O/r02_bench_c2_gates.json 2>&1
$B --config C4 --steps 20 --no-cpu-baseline > $O/r02_bench_c4.json 2>&1
$B --config C4 --steps 20 --round rtz --no-cpu-baseline > $O/r02_bench_c4_rtz.json 2>&1
$B --config C4 --steps 10 --kernel gates --no-cpu-baseline > $O/r02_bench_c4_gates.json 2>&1
$B --config C5 --sweep --steps 10 > $O/r02_bench_c5_sweep.json 2>&1
$B --config C5 --sweep --steps 10 --round rtz > $O/r02_bench_c5_sweep_rtz.json 2>&1
$B --config C5 --sweep --steps 5 --extended 1 > $O/r02_bench_c5_sweep_extended.json 2>&1
python tools/edge_bench.py > $O/r02_edge_kernels.txt 2>&1
python tools/edge_bench.py --flush read > $O/r02_edge_kernels_readflush.txt 2>&1
export HOBF_OVERSUBSCRIBE=1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > $O/r02_split_c3_n2.json 2> $O/r02_split_c3_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29513 bench.py --config C4 --gpus 8 --steps 2 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > $O/r02_split_c4_n8.json 2> $O/r02_split_c4_n8.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --config C2 --gpus 2 --steps 3 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > $O/r02_split_c2_n2.json 2> $O/r02_split_c2_n2.err
unset HOBF_OVERSUBSCRIBE
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv"
ncu $M --log-file $O/r02_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sass > /dev/null 2>&1
ncu $M --log-file $O/r02_launches_c4.csv python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sass > /dev/null 2>&1
ncu $M --log-file $O/r02_launches_mobdw.csv python bench.py --config MOBDW --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sass > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on -f"
cap() {  # name kernel-regex args...
  name=$1; k=$2; shift 2
  timeout 300 $N -k regex:$k --launch-skip 2 --launch-count 1 -o /tmp/$name python tools/ncu_target.py "$@" > $O/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep "$name: $*" > $O/$name.txt 2>&1
}
cap r02_ncu_c3_conv conv_tab --config C3
cap r02_ncu_c4_conv conv_tab --config C4
cap r02_ncu_c3_quant quantize_acts --config C3
cap r02_ncu_c4_quant quantize_acts --config C4
cap r02_ncu_mobdw_dw conv_dw --config MOBDW
python tools/sass_loop_stats.py e5m3 conv_tab_smem > $O/r02_sass_e5m3_conv_loops.txt 2>&1
ls $O | wc -l
