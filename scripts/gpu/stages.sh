python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
run() { timeout 600 python scripts/kernel_bench.py --no-prefill --models llama3.2-3b --decode 2x3000 4x3000 8x3000 16x3000 2>&1 | grep decode | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  ', d['case'], 'attn %.0f GB/s (%.1f%%) %.1f us/layer' % (d['decode_attn_gbs'], 100*d['decode_attn_frac'], d['decode_attn_us_per_layer']))
"; }
for ws in "4 4" "4 8" "8 8" "4 12"; do set -- $ws; echo "warps $1 stages $2"; ASB_DECODE_WARPS=$1 ASB_DECODE_STAGES=$2 run; done
for ws in "4 4" "4 8" "8 8"; do set -- $ws; echo "no-cluster splits=16 warps $1 stages $2"; ASB_ATTN_NO_CLUSTER=1 ASB_DECODE_WARPS=$1 ASB_DECODE_STAGES=$2 run; done
