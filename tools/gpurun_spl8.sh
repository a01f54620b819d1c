W2L_LIB=abl/spl8.so timeout 600 python -m pytest tests/test_gpu_band.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1
for r in 1 2; do for v in cur spl8; do W2L_LIB=abl/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); s=d['sub']
print('$v', round(d['ms_per_step'],4), 'asg', round(s['asg_only_ms'],4), 'ctc', round(s['ctc_only_ms'],4), {k: round(v,4) for k,v in s['asg_stage_ms'].items()}, {k: round(v,4) for k,v in s['ctc_stage_ms'].items()})"; done; done
