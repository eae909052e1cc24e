timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_engine_gpu.py -x -q 2>&1 | tail -1
timeout 600 python scripts/kernel_bench.py --out gpurun_out/kernels_v6.json 2>&1 | grep prefill | cut -c1-220
timeout 600 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 --chunk=16 2>&1 | tail -1
