timeout 900 python bench.py > gpurun_out/bench_c3_u4096.json 2> gpurun_out/bench_c3_u4096.err; python3 -c "
import json
d=json.loads(open('gpurun_out/bench_c3_u4096.json').read().strip().splitlines()[-1])
print('C3', d['value'], d['e2e']['value'], json.dumps(d['policies']), d['tails_vs_mixed_fcfs'])"
timeout 2400 python scripts/policy_compare.py --config c4 --reps 2 --runs mixed_fcfs agentserve --out gpurun_out/pc_c4_u4096.json 2>&1 | tail -2 | cut -c1-330
timeout 1500 python bench.py --config c5 --steps 1 --warmup 3 --compare mixed_fcfs --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; python3 -c "
import json
d=json.loads(open('gpurun_out/bench_c5.json').read().strip().splitlines()[-1])
print('C5', d['value'], d['e2e']['value'], json.dumps(d['policies'])[:700])"
