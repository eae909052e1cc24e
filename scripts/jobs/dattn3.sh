timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_attn_paths_gpu.py -x -q 2>&1 | grep -E "^E|passed|failed" | head -5
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 2 3 4 9; do echo "== level $L"; run --models llama3.2-3b --decode 16x3000 32x3000 --level $L; done
echo "== full device C2-C5"; run
