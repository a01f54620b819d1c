set -x
for m in ctc asg both; do W2L_LIB=abl/tl.so python tools/timeline_pdl.py $m > gpurun_out/tl_$m.txt 2>&1; done
for m in both; do W2L_PDL=1 W2L_LIB=abl/tl.so python tools/timeline_pdl.py $m > gpurun_out/tl_pdl_$m.txt 2>&1; done
