timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_engine_gpu.py tests/test_decode_step_gpu.py -x -q 2>&1 | tail -1
timeout 300 python scripts/step_launches.py llama3.1-8b 64 3000 2>&1 | tail -1
timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 2>&1 | tail -1
timeout 600 python scripts/kernel_bench.py --out gpurun_out/kernels_v8.json 2>&1 | grep -E "decode|prefill" | cut -c1-230
