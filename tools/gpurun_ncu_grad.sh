# ncu --set full of the fp32 gradient kernels at the bench shape (source-level stalls)
set -x
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"grad_kernel<.*float>" -s 2 -c 2 -o gpurun_out/grad python tools/prof_chain.py all > gpurun_out/grad_ncu.log 2>&1
tail -3 gpurun_out/grad_ncu.log
