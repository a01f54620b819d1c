for lib in tlprev tlcur tlprev tlcur; do echo "== $lib"; LOOP=4 W2L_LIB=abl/$lib.so python tools/timeline_pdl.py both 2>&1 | grep -v Warn | head -9; done
