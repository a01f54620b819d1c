# ncu --set full of the fp32 chain kernels at the bench shape (source-level counts)
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"chain_kernel<float>" -s 2 -c 2 -o gpurun_out/chain python tools/prof_chain.py all > gpurun_out/chain_ncu.log 2>&1
tail -2 gpurun_out/chain_ncu.log
