# round-2 bench lines for profiles/ (one B200).  Every line: device-timed, L2 flushed.
B="python bench.py"
$B > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
$B --impl reference > gpurun_out/r02_bench_c3_reference_arm.json 2>&1
$B --round rtz --no-cpu-baseline > gpurun_out/r02_bench_c3_rtz.json 2>&1
$B --extended 1 --no-cpu-baseline > gpurun_out/r02_bench_c3_extended.json 2>&1
$B --kernel gates --no-cpu-baseline --steps 50 > gpurun_out/r02_bench_c3_gates.json 2>&1
$B --out planes --no-cpu-baseline > gpurun_out/r02_bench_c3_planes.json 2>&1
$B --relu 1 --no-cpu-baseline > gpurun_out/r02_bench_c3_relu.json 2>&1
for c in C1 C2 MOB MOBDW; do $B --config $c --steps 50 --no-cpu-baseline > gpurun_out/r02_bench_$(echo $c | tr A-Z a-z).json 2>&1; done
$B --config C4 --steps 20 --no-cpu-baseline > gpurun_out/r02_bench_c4.json 2>&1
$B --config C4 --steps 20 --round rtz --no-cpu-baseline > gpurun_out/r02_bench_c4_rtz.json 2>&1
$B --config C4 --steps 10 --kernel gates --no-cpu-baseline > gpurun_out/r02_bench_c4_gates.json 2>&1
$B --config C5 --sweep --steps 10 > gpurun_out/r02_bench_c5_sweep.json 2>&1
$B --config C5 --sweep --steps 10 --round rtz > gpurun_out/r02_bench_c5_sweep_rtz.json 2>&1
$B --config C5 --sweep --steps 5 --extended 1 > gpurun_out/r02_bench_c5_sweep_extended.json 2>&1
# strong-split correctness on ONE GPU (ranks share the device; gloo; not a scaling measurement):
# the gathered output hash must equal the N = 1 hash above
export HOBF_OVERSUBSCRIBE=1
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 3 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > gpurun_out/r02_split_c3_n$n.json 2> gpurun_out/r02_split_c3_n$n.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --config C2 --gpus $n --steps 3 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > gpurun_out/r02_split_c2_n$n.json 2> gpurun_out/r02_split_c2_n$n.err
done
# shares of C3 / C5 under the strong split (per-GPU work at N = 2, 4, 8), automatic schedule
for n in 16 8 4; do python tools/conv_variants.py --config C3 --n $n --reps 10 2>&1 | tail -1; done > gpurun_out/r02_shares_c3.txt
for n in 32 16 8; do python tools/conv_variants.py --config C5 --format e5m3 --n $n --reps 10 2>&1 | tail -1; done > gpurun_out/r02_shares_c5.txt
for n in 128 64 32; do python tools/conv_variants.py --config C4 --n $n --reps 5 2>&1 | tail -1; done > gpurun_out/r02_shares_c4.txt
