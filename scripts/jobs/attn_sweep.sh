# decode attention ring geometry on Green Context partitions (llama3.2-3b, 16 and 32 rows, ctx 3000)
for L in 2 3 4 9; do
 for ws in "4 4" "4 8" "4 12" "8 8" "8 16"; do set -- $ws
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
