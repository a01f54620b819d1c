#!/bin/bash
# One GPU session: bench line, reference arm, ncu launch list of the bench and
# one `ncu --set full` capture of the main kernels (run under gpurun).
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sub > gpurun_out/launches.csv 2> gpurun_out/launches.err
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"(chain_kernel<float|grad_kernel<[^>]*, float)" -s 4 -c 4 -o gpurun_out/full python tools/prof_chain.py all > gpurun_out/full.log 2>&1
tail -2 gpurun_out/full.log
# the kernels one criterion call enqueues, grouped by the C-ABI's NVTX range
timeout 600 ncu --nvtx --nvtx-include "w2l_ctc_loss_grad/" --metrics gpu__time_duration.sum \
  --clock-control none --csv python tools/prof_chain.py ctc > gpurun_out/nvtx_ctc.csv 2> gpurun_out/nvtx_ctc.err
