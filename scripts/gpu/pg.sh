timeout 600 python scripts/gemm_bench.py --prefill --tokens 2048 --models qwen2.5-0.5b 2>&1 | cut -c1-200
timeout 600 python scripts/gemm_bench.py --prefill --tokens 2048 --levels 7 --models qwen2.5-0.5b 2>&1 | cut -c1-200
