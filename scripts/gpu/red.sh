timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/gemm_timeline.py 64 8b 2>&1 | grep -v "epilogue threads" | cut -c1-60,150-260
timeout 600 python scripts/gemm_bench.py --tokens 8 64 --models llama3.1-8b llama3.2-3b qwen2.5-0.5b --out gpurun_out/gemm_bench_v5.json 2>&1 | cut -c1-200
for lev in 1 2 4 0; do timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1; done
timeout 900 python scripts/kernel_bench.py --out gpurun_out/kernels_v5.json 2>&1 | tail -12 | cut -c1-300
