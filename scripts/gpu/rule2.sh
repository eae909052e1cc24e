for lev in 1 2 3 4 0; do timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1; done
timeout 300 python -m pytest tests/test_forward_gpu.py tests/test_gemm_gpu.py -q -x 2>&1 | tail -1
timeout 900 python bench.py --no-cpu 2>/dev/null | cut -c1-900
