python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
run() { timeout 600 python scripts/kernel_bench.py --no-prefill --models qwen2.5-7b llama3.2-3b 2>&1 | grep decode | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  ', d['model'], d['case'], 'attn %.1f%% gemm %.1f%% step %.2f ms' % (100*d['decode_attn_frac'], 100*d['decode_gemm_frac'], d['step_ms']))
"; }
for r in 1 2; do echo "new rule"; run; echo "splits=2"; ASB_DECODE_SPLITS=2 run; done
