mkdir -p gpurun_out
for i in 1 2 3 4; do
  for cfg in "default:" "streamctc:W2L_BENCH_STREAM_CTC=1" "ctcfirst:W2L_BENCH_FIRST=ctc" "nostream:W2L_BENCH_STREAM_ASG=0"; do
    tag=${cfg%%:*}; envs=${cfg#*:}
    env $envs timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sub > gpurun_out/env_$tag$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/env_$tag$i.json')); print('$tag', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'])"
  done
done
