for env in "X=0" "X=1" "ASB_PDL_AFTER_CLUSTER=1"; do echo "== $env"; env $env timeout 600 python scripts/determinism.py llama3.2-3b 6 4 2>&1 | tail -1; done
T="tests/test_device_vs_hf_gpu.py"
for r in 1 2; do echo "== hf run $r"; timeout 900 python -m pytest -q -x -s "$T" 2>&1 | grep -E "worst|AssertionError: \(|passed|failed" | head -3; done
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for env in "X=0" "ASB_PDL_AFTER_CLUSTER=1"; do echo "=== step $env"; env $env bash -c "$(declare -f run); run --models llama3.2-3b --decode 2x3000 16x3000 32x3000; run --models qwen2.5-7b llama3.1-8b qwen2.5-0.5b"; done
