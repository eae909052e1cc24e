timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 0 1; do ASB_NO_DGEMV=$v timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -1; done
for sk in attn qkv o gate_up down norm; do echo "skip $sk"; ASB_DEBUG_SKIP=$sk timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -1; done
for v in 0 1; do ASB_NO_DGEMV=$v timeout 300 python scripts/step_launches.py llama3.2-3b 16 3000 2>&1 | tail -1; done
timeout 600 python scripts/gemm_bench.py --tokens 8 16 --models qwen2.5-0.5b llama3.2-3b --out gpurun_out/gemm_bench3.json 2>&1 | cut -c1-200
timeout 900 python bench.py --no-cpu > gpurun_out/bench_dg3.json 2> gpurun_out/bench_dg3.err; cat gpurun_out/bench_dg3.json | cut -c1-1200
