# strong split at N = 8 on ONE GPU (ranks share it; gloo): output hashes must equal the N = 1 lines
export HOBF_OVERSUBSCRIBE=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
$R --master-port 29521 bench.py --gpus 8 --steps 2 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > gpurun_out/r02_split_c3_n8.json 2> gpurun_out/r02_split_c3_n8.err
$R --master-port 29522 bench.py --config C4 --gpus 8 --steps 2 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > gpurun_out/r02_split_c4_n8.json 2> gpurun_out/r02_split_c4_n8.err
$R --master-port 29523 bench.py --config C2 --gpus 8 --steps 2 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > gpurun_out/r02_split_c2_n8.json 2> gpurun_out/r02_split_c2_n8.err
$R --master-port 29524 bench.py --config C5 --format e6m9 --gpus 8 --steps 2 --warmup 1 --no-e2e --no-sass --no-cpu-baseline > gpurun_out/r02_split_c5_e6m9_n8.json 2> gpurun_out/r02_split_c5_e6m9_n8.err
python bench.py --config C5 --format e6m9 --steps 3 --no-e2e --no-sass --no-cpu-baseline > gpurun_out/r02_bench_c5_e6m9_n1.json 2>&1
