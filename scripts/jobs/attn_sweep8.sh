run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'step %.3f' % d['step_ms_unprofiled'])
"; }
for ws in "4 6" "4 4" "2 6"; do set -- $ws
for L in 2 3 4 9; do
  echo "== warps $1 stages $2 level $L"
  ASB_DECODE_WARPS=$1 ASB_DECODE_STAGES=$2 run --models llama3.2-3b --decode 16x3000 32x3000 --level $L
done; done
echo "== attnmath"; ASB_DEBUG_SKIP=attnmath run --models llama3.2-3b --decode 16x3000 --level 2
echo "== C4/C5 full device"; run --models qwen2.5-7b llama3.1-8b qwen2.5-0.5b
timeout 900 python -m pytest tests/test_attn_paths_gpu.py tests/test_forward_gpu.py tests/test_device_vs_hf_gpu.py -q 2>&1 | tail -2
