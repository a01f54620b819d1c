CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool initcheck --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_reference_suite.py > gpurun_out/san_initcheck.log 2>&1
echo "initcheck pytest: $(grep -E 'passed|failed' gpurun_out/san_initcheck.log | tail -1) | $(grep 'ERROR SUMMARY' gpurun_out/san_initcheck.log | tail -1)"
timeout 900 $CS --tool initcheck --print-limit 20 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sub > gpurun_out/san_bench_initcheck.log 2>&1
echo "initcheck bench: $(grep 'ERROR SUMMARY' gpurun_out/san_bench_initcheck.log | tail -1)"
for r in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_x.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_x.json')); s=d['sub']
print(round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'], 'asg', round(s['asg_only_ms'],4), 'ctc', round(s['ctc_only_ms'],4))"; done
