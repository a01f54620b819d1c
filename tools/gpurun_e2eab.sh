for r in 1 2 3 4 5; do for v in prev cur; do W2L_LIB=abl/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); e=d['e2e']
print('$v', round(d['ms_per_step'],4), '%.3e'%e['value'], e['host_enqueue_ms_per_step'], '%.3e'%d['e2e_grads_to_host']['value'])"; done; done
