# prefill GEMMs per linear at the engine's 2048-token launch unit: TF/s by partition size (wave fill)
timeout 600 python scripts/gemm_bench.py --models llama3.2-3b llama3.1-8b --tokens 2048 3000 --levels 0 5 6 7 --prefill --iters 20 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'][:10], d['linear'], 'T', d['T'], 'sms', d['sms'], '%.0f TF/s' % d.get('tflops',0))
"
