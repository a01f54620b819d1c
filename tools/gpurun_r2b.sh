# parity suite + bench + reference-suite on one box
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --no-cpu-baseline --no-sub > gpurun_out/bench2.json 2>> gpurun_out/bench.err
tail -3 gpurun_out/smoke.log gpurun_out/gputest.log
python - <<'PY'
import json
for f in ["gpurun_out/bench.json","gpurun_out/bench2.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["ms_per_step"], d["e2e"]["value"], d.get("sub",{}).get("asg_only_ms"), d.get("sub",{}).get("ctc_only_ms"))
    except Exception as e: print(f, "ERR", e)
PY
