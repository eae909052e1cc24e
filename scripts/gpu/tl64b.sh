timeout 300 python scripts/gemm_timeline.py 64 8b 2>&1 | cut -c1-40,150-330
