# Cross-kernel L2 prefetch of the next decode linear's first ring fill (ASB_TG_L2PF=1) vs off: decode step by partition level
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer' % d['decode_attn_us_per_layer'], 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 3 4 7 9; do
  for pf in 0 1; do echo "== level $L pf $pf"; ASB_TG_L2PF=$pf run --models llama3.2-3b --decode 8x3000 16x3000 --level $L; done
done
for pf in 0 1; do echo "== 8B level 4 / 9 pf $pf"; ASB_TG_L2PF=$pf run --models llama3.1-8b --decode 16x3000 --level 4; ASB_TG_L2PF=$pf run --models llama3.1-8b --decode 16x3000 --level 9; done
ASB_TG_L2PF=1 timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_determinism_gpu.py -x -q 2>&1 | tail -1
