for L in 2 3 4 9; do
 for ws in "4 4" "4 8"; do set -- $ws
  echo "== level $L warps $1 stages $2"
  ASB_DECODE_WARPS=$1 ASB_DECODE_STAGES=$2 timeout 300 python scripts/kernel_bench.py --models llama3.2-3b --no-prefill --decode 16x3000 32x3000 --level $L --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f ms' % d['step_ms_unprofiled'])
"
 done
done
timeout 600 python -m pytest tests/test_attn_paths_gpu.py tests/test_forward_gpu.py -q 2>&1 | tail -2
