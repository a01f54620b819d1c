#!/bin/bash
# One GPU session at HEAD: smoke, GPU parity suite, bench line + reference arm,
# ncu launch list of the bench and one `ncu --set full` capture of the chains/grads.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
bash tools/profile_round.sh
tail -3 gpurun_out/smoke.log gpurun_out/gputest.log
cat gpurun_out/bench.json gpurun_out/ref.json
