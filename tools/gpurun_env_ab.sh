#!/bin/bash
# A/B of bench.py schedule variants: each "tag:lib:ENV=..." runs with abl/<lib>.so
# and the given environment; alternating rounds, device ms and e2e frames/s.
#   bash tools/gpurun_env_ab.sh <rounds> "default:base:" "sctc:base:W2L_BENCH_STREAM_CTC=1" ...
mkdir -p gpurun_out
R=$1; shift
for i in $(seq 1 $R); do
  for cfg in "$@"; do
    tag=${cfg%%:*}; rest=${cfg#*:}; lib=${rest%%:*}; envs=${rest#*:}
    env W2L_LIB=abl/$lib.so $envs timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/env_$tag$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/env_$tag$i.json')); print('$tag', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'], '%.3e'%d['e2e_grads_to_host']['value'])"
  done
done
