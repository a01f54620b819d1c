for r in 1 2 3; do for f in ctc asg; do W2L_BENCH_FIRST=$f timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_o.json 2>gpurun_out/ab_o.err; python -c "
import json; d=json.load(open('gpurun_out/ab_o.json')); e=d['e2e']; g=d['e2e_grads_to_host']
print('first=$f', round(d['ms_per_step'],4), '%.3e'%e['value'], e['host_enqueue_ms_per_step'], '%.3e'%g['value'], g['host_enqueue_ms_per_step'])" || tail -3 gpurun_out/ab_o.err; done; done
