python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
run() { timeout 600 python scripts/kernel_bench.py --no-prefill --models llama3.2-3b --decode 24x3000 32x3000 48x3000 2>&1 | grep decode | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  ', d['case'], 'attn %.0f GB/s (%.1f%%) %.1f us/layer' % (d['decode_attn_gbs'], 100*d['decode_attn_frac'], d['decode_attn_us_per_layer']))
"; }
for sp in 2 3 4; do echo "cluster splits=$sp"; ASB_DECODE_SPLITS=$sp run; echo "no-cluster splits=$sp"; ASB_ATTN_NO_CLUSTER=1 ASB_DECODE_SPLITS=$sp run; done
