# page-granular decode attention (one 32 KiB TMA per K|V block): correctness then partition rates
timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_attn_paths_gpu.py tests/test_engine_gpu.py -x -q 2>&1 | grep -E "^E|passed|failed" | head -8
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 1 2 4 9; do echo "== level $L"; run --models llama3.2-3b --decode 16x3000 32x3000 --level $L; done
echo "== attnmath level 2"; ASB_DEBUG_SKIP=attnmath run --models llama3.2-3b --decode 16x3000 32x3000 --level 2
echo "== full device C2-C5"; run
timeout 600 python scripts/gemm_bench.py --models llama3.2-3b --tokens 16 32 --levels 1 2 4 0 2>&1 | tail -40
timeout 1500 python -m pytest tests/test_forward_c4c5_gpu.py -x -q -s 2>&1 | grep -E "near-ties|passed|failed|Error" | head -20
