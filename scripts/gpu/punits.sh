python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
true
for v in 1 0 1 0 1 0; do echo "units=$v"; ASB_PREFILL_UNITS=$v timeout 300 python scripts/kernel_bench.py --models qwen2.5-0.5b --out /tmp/kb.json 2>&1 | grep prefill | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  ', d['case'], 'attn %.1f TF/s gemm %.1f TF/s forward %.3f ms' % (d['prefill_attn_tflops'], d['prefill_gemm_tflops'], d['forward_ms']))
"; done
