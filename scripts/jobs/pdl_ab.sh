run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for env in "X=0" "ASB_ATTN_NO_CLUSTER=1" "ASB_GEMM_SPLITS=1" "ASB_ATTN_NO_CLUSTER=1 ASB_GEMM_SPLITS=1"; do echo "=== step $env"; env $env bash -c "$(declare -f run); run --models llama3.2-3b --decode 2x3000 16x3000 32x3000; run --models llama3.2-3b --decode 16x3000 --level 4; run --models qwen2.5-7b llama3.1-8b"; done
for env in "ASB_ATTN_NO_CLUSTER=1 ASB_GEMM_SPLITS=1"; do echo "== det $env"; env $env timeout 600 python scripts/determinism.py llama3.2-3b 4 4 2>&1 | tail -1; done
