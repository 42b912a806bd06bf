(time python -m pytest tests -m gpu -x -q) > gpurun_out/s4_gputest.log 2>&1; tail -3 gpurun_out/s4_gputest.log
B="python bench.py --no-cpu-baseline"
$B > gpurun_out/s4_bench_c3.json 2>&1
$B --config C4 --steps 20 > gpurun_out/s4_bench_c4.json 2>&1
$B --config MOBDW --steps 50 > gpurun_out/s4_bench_mobdw.json 2>&1
$B --config MOB --steps 50 > gpurun_out/s4_bench_mob.json 2>&1
$B --kernel gates --steps 50 > gpurun_out/s4_bench_c3_gates.json 2>&1
for f in gpurun_out/s4_bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', '%.4g'%d['value'], d['ms_per_step'], r['frac'], r.get('gates_per_32lane_mac'))"; done
