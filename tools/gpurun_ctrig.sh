# CTC gradient streamed with a late trigger (its grid queued before ASG's last gradient CTAs)
for r in 1 2 3; do for cfg in "cur 0" "cur 1" "c34 1" "c910 1"; do set -- $cfg
W2L_LIB=abl/$1.so W2L_BENCH_STREAM_CTC=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_t.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_t.json'))
print('$1 sc=$2', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'])"; done; done
