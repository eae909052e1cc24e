# tgemv at 17-32 tokens with 16 consumer warps vs the tcgen05 swap-AB kernel
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -1
timeout 600 python scripts/gemm_bench.py --models llama3.2-3b llama3.1-8b --tokens 24 32 --levels 1 2 3 4 0 --paths 1 3 --iters 30 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'][:10], d['linear'], 'T', d['T'], 'sms', d['sms'], 'tc %.0f' % d.get('p1_gbs',0), 'tg %.0f' % d.get('p3_gbs',0), 'tg/tc %.2f' % (d.get('p3_gbs',0)/max(1,d.get('p1_gbs',1))))
"
