nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc scripts/probes/tma_pair.cu paper_2603_10342_b200/csrc/tmap.cpp -lcuda -o /tmp/tma_pair && timeout 120 /tmp/tma_pair | grep packed
for skip in none tgmath; do echo "== skip $skip"; ASB_DEBUG_SKIP=$skip timeout 300 python scripts/gemm_bench.py --models llama3.2-3b --linears gate_up qkv --tokens 16 --levels 1 2 4 0 --paths 3 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['linear'], 'T', d['T'], 'sms', d['sms'], 'tgemv %.0f GB/s' % d.get('p3_gbs',0), '(%.0f GB/s/SM)' % (d.get('p3_gbs',0)/d['sms']))
"; done
