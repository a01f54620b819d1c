for r in 1 2 3; do for kb in 80 64 100; do W2L_CHAIN_SMEM_KB=$kb timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_s.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_s.json'))
print('smem=$kb', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'])"; done; done
