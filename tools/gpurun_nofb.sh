for r in 1 2 3; do for v in 0 1; do W2L_BENCH_NOFB=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_f.json'))
print('nofb=$v', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'])"; done; done
