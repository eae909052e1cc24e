timeout 600 python scripts/gemm_bench.py --tokens 8 16 32 --sms 0 32 --out gpurun_out/gemm_bench.json 2>&1 | tail -70
