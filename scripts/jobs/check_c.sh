run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 2 3 4 9; do run --models llama3.2-3b --decode 16x3000 32x3000 --level $L; ASB_DEBUG_SKIP=attnmath run --models llama3.2-3b --decode 16x3000 --level $L; done > gpurun_out/check_c_kern.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/check_c_tests.txt 2>&1; tail -2 gpurun_out/check_c_tests.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; tail -c 600 gpurun_out/bench_c.json
