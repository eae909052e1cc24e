for lev in 1 2 4 0; do for v in 0 1; do ASB_NO_DGEMV=$v timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1; done; done
timeout 300 python -m pytest tests/test_forward_gpu.py -q -x 2>&1 | tail -1
