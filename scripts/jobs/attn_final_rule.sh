# Decode split rules final (one wave pow2; persistent 1 split): step by level, attention-path parity, C3 policy comparison (10 reps)
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 3 4 5 6 7 9; do echo "== level $L"; run --models llama3.2-3b --decode 4x3000 8x3000 16x3000 24x3000 32x3000 --level $L; done
timeout 1200 python -m pytest tests/test_attn_paths_gpu.py -x -q 2>&1 | tail -1
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve agentserve:dt=50 agentserve:thigh=0.85 mixed_fcfs --out gpurun_out/pc_c3_attnrule.json 2>&1 | tail -1 | cut -c1-200
