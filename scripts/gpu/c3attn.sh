for sp in 16 1 3 4; do echo "max_splits=$sp"; ASB_DECODE_MAX_SPLITS=$sp timeout 600 python scripts/kernel_bench.py --models llama3.2-3b qwen2.5-7b 2>&1 | grep decode | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['model'], d['case'], 'attn %.0f GB/s (%.1f%%) %.1f us/layer' % (d['decode_attn_gbs'], 100*d['decode_attn_frac'], d['decode_attn_us_per_layer']))
"; done
timeout 900 python bench.py --no-cpu 2>/dev/null | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['latency_ms']['tpot'], d['roofline'])"
