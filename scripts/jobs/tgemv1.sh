timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q -k "3-" 2>&1 | grep -E "^E|passed|failed" | head -8
timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_engine_gpu.py tests/test_forward_c4c5_gpu.py -x -q -s 2>&1 | grep -E "^E|passed|failed|near-ties" | head -12
timeout 600 python scripts/gemm_bench.py --models llama3.2-3b --tokens 16 32 --levels 1 2 3 4 0 --paths 1 3 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['linear'], 'T', d['T'], 'sms', d['sms'], 'tcgen05 %.0f GB/s' % d.get('p1_gbs',0), 'tgemv %.0f GB/s' % d.get('p3_gbs',0), '(%.0f GB/s/SM)' % (d.get('p3_gbs',0)/d['sms']))
"
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 1 2 3 4 9; do echo "== level $L"; run --models llama3.2-3b --decode 16x3000 32x3000 --level $L; done
echo "== full device C2-C5"; run
