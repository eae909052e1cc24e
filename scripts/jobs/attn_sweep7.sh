for skip in "" "attnmath"; do
for L in 2 3 4 9; do
  echo "== skip=$skip level $L"
  ASB_DEBUG_SKIP=$skip timeout 300 python scripts/kernel_bench.py --models llama3.2-3b --no-prefill --decode 16x3000 32x3000 --level $L --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'step %.3f' % d['step_ms_unprofiled'])
"
done; done
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
