# streamed gradient warps pausing per frame while their chains run
W2L_LIB=abl/y300.so timeout 600 python -m pytest tests/test_gpu_band.py -q -p no:cacheprovider 2>&1 | tail -1
for r in 1 2 3; do for v in cur y100 y300 y1000; do W2L_LIB=abl/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/ab_y.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_y.json'))
print('$v', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'])"; done; done
