# the scheduled step (ASG first): timeline, bench line, A/B vs CTC first
LOOP=4 W2L_LIB=abl/tl.so python tools/timeline_pdl.py both 2>&1 | grep -v Warn | sed -n 1,16p | grep -v "slowest\|pair"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_sched.json 2>gpurun_out/bench_sched.err; tail -c 600 gpurun_out/bench_sched.json
for r in 1 2 3; do for f in ctc asg; do W2L_BENCH_FIRST=$f timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_o.json 2>gpurun_out/ab_o.err; python -c "
import json; d=json.load(open('gpurun_out/ab_o.json'))
print('first=$f', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'], '%.3e'%d['e2e_grads_to_host']['value'], d['config']['schedule'])" || tail -3 gpurun_out/ab_o.err; done; done
