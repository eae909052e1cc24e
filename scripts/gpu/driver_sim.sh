set -o pipefail
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ds_build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ds_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/ds_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ds_tests.log
timeout 900 python bench.py --impl reference > gpurun_out/ds_ref.json 2> gpurun_out/ds_ref.err; echo ref=$?
timeout 900 python bench.py > gpurun_out/ds_bench.json 2> gpurun_out/ds_bench.err; echo bench=$?
python3 -c "
import json
b=json.loads(open('gpurun_out/ds_bench.json').read().strip().splitlines()[-1]); r=json.loads(open('gpurun_out/ds_ref.json').read().strip().splitlines()[-1])
print('bench', b['value'], b['unit'], 'e2e', b['e2e']['value'], 'tpot', b.get('latency_ms',{}).get('tpot'), 'clocks', b.get('clocks'))
print('roofline', b['roofline'])
print('ref', r.get('value'), r.get('unit'), r.get('cpu_baseline'))
"
