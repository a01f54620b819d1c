# CTC stream priority / streamed CTC gradient in the two-criteria step
for cfg in "0 0" "-1 0" "0 1" "-1 1"; do set -- $cfg
echo "== prio=$1 stream_ctc=$2"; W2L_BENCH_PRIO=$1 W2L_BENCH_STREAM_CTC=$2 LOOP=4 W2L_LIB=abl/tl.so python tools/timeline_pdl.py both 2>&1 | grep -v Warn | sed -n 1,16p | grep "call\|chain  \|grad  "; done
for r in 1 2 3; do for cfg in "0 0" "-1 0" "0 1" "-1 1"; do set -- $cfg
W2L_BENCH_PRIO=$1 W2L_BENCH_STREAM_CTC=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_p.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_p.json'))
print('prio=$1 sc=$2', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'])"; done; done
