# stagger order and which criterion streams its gradient
for r in 1 2 3; do for cfg in "0 1 0" "1 1 0" "1 0 1" "1 1 1" "1 0 0"; do set -- $cfg
W2L_BENCH_ASG_FIRST=$1 W2L_BENCH_STREAM_ASG=$2 W2L_BENCH_STREAM_CTC=$3 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_o.json 2>gpurun_out/ab_o.err; python -c "
import json; d=json.load(open('gpurun_out/ab_o.json'))
print('asg_first=$1 sa=$2 sc=$3', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'])" || tail -3 gpurun_out/ab_o.err; done; done
