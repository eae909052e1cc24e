# One-wave decode split rule: decode step by level, attention-path + forward parity tests, C3 AgentServe vs FCFS (10 reps)
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 3 4 5 6 7 8 9; do echo "== level $L"; run --models llama3.2-3b --decode 4x3000 8x3000 16x3000 24x3000 --level $L; done
echo "== C4/C5 full device"; run --models qwen2.5-7b llama3.1-8b
timeout 1200 python -m pytest tests/test_attn_paths_gpu.py tests/test_forward_gpu.py tests/test_forward_c4c5_gpu.py tests/test_determinism_gpu.py -x -q 2>&1 | tail -1
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve agentserve:dt=50 --out gpurun_out/pc_c3_onewave.json 2>&1 | tail -1 | cut -c1-200
