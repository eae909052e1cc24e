# tgemv two-phase plan (whole tiles in full waves + remainder tiles split over the grid) vs uniform (ASB_TGEMV_UNIFORM=1): parity, decode step by level, C3 policy comparison
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_forward_gpu.py tests/test_engine_gpu.py tests/test_determinism_gpu.py -x -q 2>&1 | tail -1
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer' % d['decode_attn_us_per_layer'], 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 3 5 6 7 8; do for u in 0 1; do echo "== level $L uniform=$u"; if [ $u = 1 ]; then export ASB_TGEMV_UNIFORM=1; else unset ASB_TGEMV_UNIFORM; fi; run --models llama3.2-3b llama3.1-8b --decode 8x3000 16x3000 --level $L; done; done
unset ASB_TGEMV_UNIFORM
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve --out gpurun_out/pc_c3_twophase.json 2>&1 | tail -1 | cut -c1-200
