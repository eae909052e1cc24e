timeout 300 python scripts/gemm_timeline.py 64 8b 2>&1 | tail -8
