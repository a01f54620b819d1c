# usage: bash tools/gpurun_ab.sh A B [rounds]  (abl/A.so vs abl/B.so): parity of B, then A/B bench
A=$1; B=$2; R=${3:-3}
W2L_LIB=abl/$B.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_$B.log 2>&1; echo "pytest($B) rc=$?" >> gpurun_out/gputest_$B.log
tail -3 gpurun_out/gputest_$B.log
bash tools/ab.sh abl/$A.so abl/$B.so $R 2>&1
for tag in $A $B; do
W2L_LIB=abl/$tag.so timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/sub_$tag.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/sub_$tag.json')); s=d['sub']; print('$tag', s['asg_only_ms'], s['ctc_only_ms'], s['asg_stage_ms'], s['ctc_stage_ms'], {k:(v['asg_fallbacks'],v['ctc_fallbacks'],round(v['asg_ms'],3),round(v['ctc_ms'],3)) for k,v in s['peaky_emissions'].items()})"
done
