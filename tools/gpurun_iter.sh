# one iteration: GPU parity suite, bench line, ncu of the fp32 gradient kernels
set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.json 2>gpurun_out/bench_iter.err
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:"grad_kernel<.*float>" -s 2 -c 2 -o gpurun_out/grad python tools/prof_chain.py all > gpurun_out/grad_ncu.log 2>&1
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_iter.json").read().strip().splitlines()[-1]); s=d.get("sub",{})
print(round(d["ms_per_step"],4), round(d["e2e"]["value"]/1e6,1), s.get("asg_only_ms"), s.get("ctc_only_ms"), s.get("asg_stage_ms"), s.get("ctc_stage_ms"), s.get("fp32_guard_fallbacks"), {k:(round(v["asg_ms"],3),round(v["ctc_ms"],3),v["asg_fallbacks"],v["ctc_fallbacks"]) for k,v in s.get("peaky_emissions",{}).items()})
PY
