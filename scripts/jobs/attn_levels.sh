# Decode attention at 80-112 SM partitions is slower than at 64 SMs (B=16 ctx 3000: 60/52/53 vs 37 us/layer): forced split counts and the persistent kernel by level
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 4 5 7 9; do
  echo "== level $L default"; run --models llama3.2-3b --decode 8x3000 16x3000 32x3000 --level $L
  for sp in 1 2 3 4; do echo "-- splits $sp"; ASB_DECODE_SPLITS=$sp run --models llama3.2-3b --decode 8x3000 16x3000 --level $L; done
  echo "-- persist"; ASB_DECODE_PERSIST=1 run --models llama3.2-3b --decode 8x3000 16x3000 32x3000 --level $L
  echo "-- no cluster"; ASB_ATTN_NO_CLUSTER=1 run --models llama3.2-3b --decode 8x3000 16x3000 --level $L
done
