timeout 600 python scripts/gemm_bench.py --tokens 8 --levels 1 2 4 --models qwen2.5-0.5b --out gpurun_out/gemm_bench_part.json 2>&1 | cut -c1-220
for lev in 1 2 4; do for v in 0 1; do ASB_NO_DGEMV=$v timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 --level=$lev 2>&1 | tail -1; done; done
for lev in 1 2; do ASB_DEBUG_SKIP=attn timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 --level=$lev 2>&1 | tail -1; done
