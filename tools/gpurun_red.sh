W2L_LIB=abl/cur.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
for r in 1 2 3; do for v in prev cur; do W2L_LIB=abl/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); s=d['sub']
print('$v', round(d['ms_per_step'],4), 'asg', round(s['asg_only_ms'],4), 'ctc', round(s['ctc_only_ms'],4), 'asg grad', round(s['asg_stage_ms']['grad'],4))"; done; done
W2L_LIB=abl/cur.so timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,gpu__time_duration.sum -k regex:"asg_grad_kernel<[^>]*, float" -s 2 -c 1 python tools/prof_chain.py asg 2>&1 | grep -E "conflicts|duration" | head -3
