timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_full.log 2>&1; tail -3 gpurun_out/gputest_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c3_final4.json 2> gpurun_out/bench_c3_final4.err; python3 -c "
import json
d=json.loads(open('gpurun_out/bench_c3_final4.json').read().strip().splitlines()[-1])
print('C3', d['value'], d['e2e']['value'], json.dumps(d['policies']), d['tails_vs_mixed_fcfs'], d['roofline']['frac'], d.get('decode_attn'))"
