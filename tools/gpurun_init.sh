timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log; tail -2 gpurun_out/gputest.log
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_reference_suite.py > gpurun_out/san_initcheck.log 2>&1
echo "initcheck pytest: $(grep -E 'passed|failed' gpurun_out/san_initcheck.log | tail -1) | $(grep 'ERROR SUMMARY' gpurun_out/san_initcheck.log | tail -1)"
