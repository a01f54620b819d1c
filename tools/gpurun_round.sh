#!/bin/bash
# One GPU session at HEAD: smoke, GPU parity suite, bench line + reference arm,
# ncu launch list of the bench, one `ncu --set full` capture of the fp32 chains
# and gradients, and the CTA timelines of a call (timeline build in abl/tl.so).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
bash tools/profile_round.sh
if [ -f abl/tl.so ]; then for m in asg ctc; do W2L_LIB=abl/tl.so python tools/timeline_pdl.py $m > gpurun_out/tl_$m.txt 2>&1; done; LOOP=4 W2L_LIB=abl/tl.so python tools/timeline_pdl.py both > gpurun_out/tl_both.txt 2>&1; fi
tail -n 3 gpurun_out/smoke.log gpurun_out/gputest.log
cat gpurun_out/bench.json gpurun_out/ref.json
