for r in 1 2 3 4; do for v in 0 1; do W2L_BENCH_CTC_GRAD_PRIO=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_g.json 2>gpurun_out/ab_g.err; python -c "
import json; d=json.load(open('gpurun_out/ab_g.json'))
print('ctc_grad_prio=$v', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'])" || tail -3 gpurun_out/ab_g.err; done; done
