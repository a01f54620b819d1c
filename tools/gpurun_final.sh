# asg_final: 512 threads with 16/8/4 partials in flight per entry vs HEAD (256 threads)
W2L_LIB=abl/cur.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for r in 1 2 3; do for v in prev cur fc8 fc4; do W2L_LIB=abl/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); s=d['sub']
print('$v', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'], 'asg', round(s['asg_only_ms'],4), 'ctc', round(s['ctc_only_ms'],4), {k: round(v,4) for k,v in s['asg_stage_ms'].items()})"; done; done
