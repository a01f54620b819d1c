python tools/dbg_flush.py > gpurun_out/dbg.log 2>&1
W2L_NO_PDL=1 python tools/dbg_flush.py > gpurun_out/dbg_nopdl.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_pdl$i.json 2>/dev/null
W2L_NO_PDL=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_nopdl$i.json 2>/dev/null
done
W2L_NO_PDL=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_nopdl.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sub > /dev/null 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_*pdl*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); s=d.get("sub",{}); print(f, round(d["ms_per_step"],4), round(d["e2e"]["value"]/1e6,1), s.get("asg_only_ms"), s.get("ctc_only_ms"), s.get("asg_stage_ms"), s.get("ctc_stage_ms"))
    except Exception as e: print(f, "ERR", e)
PY
