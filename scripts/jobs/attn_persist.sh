# Persistent decode attention split count by level (B=24/32 rows ctx 3000, more (row, head) items than one wave); default vs forced
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 2 3 4 5; do
  echo "== level $L default"; run --models llama3.2-3b --decode 4x3000 8x3000 24x3000 32x3000 --level $L
  for sp in 1 2 3 4 6 8; do echo "-- persist splits $sp"; ASB_DECODE_PERSIST_SPLITS=$sp run --models llama3.2-3b --decode 24x3000 32x3000 --level $L; done
done
for L in 6 7 8 9; do echo "== level $L default"; run --models llama3.2-3b --decode 4x3000 8x3000 --level $L; done
