for m in asg ctc; do W2L_LIB=abl/tl.so python tools/timeline_pdl.py $m > gpurun_out/tl_$m.txt 2>&1; done
