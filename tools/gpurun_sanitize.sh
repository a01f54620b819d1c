# compute-sanitizer memcheck / initcheck / synccheck over the GPU suite and the bench configuration
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck initcheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --deselect tests/test_reference_suite.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool pytest: $(grep -E 'passed|failed' gpurun_out/san_$tool.log | tail -1) | $(grep 'ERROR SUMMARY' gpurun_out/san_$tool.log | tail -1)"
done
for tool in memcheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sub > gpurun_out/san_bench_$tool.log 2>&1
  echo "$tool bench: $(grep 'ERROR SUMMARY' gpurun_out/san_bench_$tool.log | tail -1)"
done
# racecheck (shared-memory hazards) over the band-limited gradient tests (slow: one file)
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_band.py -q -p no:cacheprovider > gpurun_out/san_racecheck.log 2>&1
echo "racecheck band tests: $(grep -E 'passed|failed' gpurun_out/san_racecheck.log | tail -1) | $(grep 'RACECHECK SUMMARY\|ERROR SUMMARY' gpurun_out/san_racecheck.log | tail -1)"
