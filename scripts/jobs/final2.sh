timeout 2400 python scripts/policy_compare.py --config c3 --reps 5 --runs mixed_fcfs agentserve --out gpurun_out/pc_c3_final2.json 2>&1 | tail -2 | cut -c1-500
timeout 900 python bench.py > gpurun_out/bench_c3_final2.json 2> gpurun_out/bench_c3_final2.err; python3 -c "
import json
d=json.loads(open('gpurun_out/bench_c3_final2.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], json.dumps(d['policies']), d['tails_vs_mixed_fcfs'])"
