# ncu launch list (per-kernel durations) of a short bench run + bench line
timeout 300 python bench.py --no-cpu-baseline --no-sub > gpurun_out/bench_l.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_l.json')); print('bench', d['ms_per_step'], d['e2e']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sub > gpurun_out/launches.csv 2> gpurun_out/launches.err
