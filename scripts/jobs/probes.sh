# Small-partition decode: per-CTA TMA streaming ceiling and decode attention/GEMM at 16-64 SMs,
# with the consumer math removed (attnmath) and deeper rings, to separate latency from issue.
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc \
  scripts/probes/tma_stride.cu paper_2603_10342_b200/csrc/tmap.cpp -lcuda -o /tmp/tma_stride && /tmp/tma_stride
run() { timeout 300 python scripts/kernel_bench.py --no-prefill "$@" --out /tmp/k.json 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['model'], d['case'], 'sms', d['sms'], 'attn %.1f us/layer %.0f GB/s' % (d['decode_attn_us_per_layer'], d['decode_attn_gbs']), 'gemm %.0f GB/s' % d['decode_gemm_gbs'], 'step %.3f' % d['step_ms_unprofiled'])
"; }
for L in 1 2 4 9; do
  echo "== default level $L"; run --models llama3.2-3b --decode 16x3000 32x3000 --level $L
  echo "== attnmath level $L"; ASB_DEBUG_SKIP=attnmath run --models llama3.2-3b --decode 16x3000 32x3000 --level $L
  echo "== stages8 level $L"; ASB_DECODE_STAGES=8 run --models llama3.2-3b --decode 16x3000 32x3000 --level $L
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc scripts/probes/tma_pair.cu paper_2603_10342_b200/csrc/tmap.cpp -lcuda -o /tmp/tma_pair && /tmp/tma_pair
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc scripts/probes/hmma.cu -o /tmp/hmma && /tmp/hmma
