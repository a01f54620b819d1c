for r in 1 2 3; do for v in 0 1; do W2L_CHAIN_PDL=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_c.json')); s=d['sub']
print('chain_pdl=$v', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'], 'asg', round(s['asg_only_ms'],4), 'ctc', round(s['ctc_only_ms'],4))"; done; done
