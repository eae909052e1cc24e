timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_attn_paths_gpu.py -x -q 2>&1 | grep -E "^E|passed|failed" | head -5
timeout 600 python scripts/kernel_bench.py --models qwen2.5-0.5b llama3.2-3b qwen2.5-7b llama3.1-8b --no-decode --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'gemm %.0f TF/s' % d['prefill_gemm_tflops'], 'attn %.0f TF/s' % d['prefill_attn_tflops'], 'fwd %.2f ms' % d['forward_ms'])
"
