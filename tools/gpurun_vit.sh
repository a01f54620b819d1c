# chunked parallel Viterbi traceback: bit-exact tests, then time vs HEAD
W2L_LIB=abl/cur.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_eval.py -q -p no:cacheprovider -k "viterbi or Viterbi or c4 or eval" 2>&1 | tail -2
for r in 1 2 3; do for v in prev cur; do echo -n "$v "; W2L_LIB=abl/$v.so python tools/vit_time.py 2>&1 | tail -1; done; done
