set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -5 gpurun_out/gputest.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_pdl$i.json 2>/dev/null
W2L_NO_PDL=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_nopdl$i.json 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_*pdl*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); s=d.get("sub",{})
        print(f, round(d["ms_per_step"],4), round(d["e2e"]["value"]/1e6,1), s.get("asg_only_ms"), s.get("ctc_only_ms"), s.get("fp32_guard_fallbacks"), {k:(round(v["asg_ms"],3),round(v["ctc_ms"],3)) for k,v in s.get("peaky_emissions",{}).items()})
    except Exception as e: print(f, "ERR", e)
PY
