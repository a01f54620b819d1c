#!/bin/bash
# A/B of library variants built by tools/ab_flags.sh into abl/<tag>.so:
#   bash tools/gpurun_ab_variants.sh "<test-tag>" <rounds> tag1 tag2 ...
# runs the GPU suite with abl/<test-tag>.so, then alternates bench.py runs.
mkdir -p gpurun_out
TT=$1; R=$2; shift 2
if [ -n "$TT" ]; then
  W2L_LIB=abl/$TT.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_$TT.log 2>&1
  echo "tests($TT): $(tail -1 gpurun_out/gputest_$TT.log)"
fi
for i in $(seq 1 $R); do
  for v in "$@"; do
    W2L_LIB=abl/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v$i.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_$v$i.json')); s=d['sub']
print('$v', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'], 'asg', round(s['asg_only_ms'],4), 'ctc', round(s['ctc_only_ms'],4), 'grad', round(s['asg_stage_ms']['grad'],4), round(s['ctc_stage_ms']['grad'],4))"
  done
done
