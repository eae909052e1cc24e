python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
for sp in 16 1; do echo "max_splits=$sp"; ASB_DECODE_MAX_SPLITS=$sp timeout 600 python scripts/kernel_bench.py --no-prefill --models llama3.2-3b --decode 4x3000 8x3000 16x3000 24x3000 48x3000 64x3000 2>&1 | grep decode | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['model'], d['case'], 'attn %.0f GB/s (%.1f%%) %.1f us/layer' % (d['decode_attn_gbs'], 100*d['decode_attn_frac'], d['decode_attn_us_per_layer']))
"; done
