timeout 900 python scripts/gemm_bench.py --models qwen2.5-0.5b llama3.2-3b llama3.1-8b --tokens 8 16 --levels 1 2 3 4 0 --paths 1 2 3 --iters 30 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'][:10], d['linear'], 'T', d['T'], 'sms', d['sms'], 'tc %.0f' % d.get('p1_gbs',0), 'dg %.0f' % d.get('p2_gbs',0), 'tg %.0f' % d.get('p3_gbs',0))
"
