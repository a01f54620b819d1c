for dl in 0 0 40000 40000; do echo "== delay $dl"; LOOP=4 TL_ASG_DELAY=$dl W2L_LIB=abl/tlcur.so python tools/timeline_pdl.py both 2>&1 | grep -v Warn | sed -n 1,9p | grep -v "slowest\|pair"; done
