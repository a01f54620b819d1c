# A/B timing of two builds of the library on the same box:
#   bash tools/ab.sh <libA.so> <libB.so> [rounds]
# alternates bench.py runs (device ms/step, e2e frames/s, ASG/CTC grad ms).
A=$1; B=$2; R=${3:-3}
for i in $(seq 1 $R); do
  for tag in A B; do
    if [ $tag = A ]; then L=$A; else L=$B; fi
    W2L_LIB=$L timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$tag$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$tag$i.json')); s=d['sub']; print('$tag', round(d['ms_per_step'],4), '%.3e'%d['e2e']['value'], round(s['asg_stage_ms']['grad'],4), round(s['ctc_stage_ms']['grad'],4), round(s['asg_stage_ms']['chain'],4), round(s['ctc_stage_ms']['chain'],4))"
  done
done
