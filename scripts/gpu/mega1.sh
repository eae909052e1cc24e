timeout 300 python -m pytest tests/test_decode_step_gpu.py -x -q -s 2>&1 | tail -15
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for lev in 1 2 0; do for v in 0 1; do ASB_NO_MEGA=$v timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 --level=$lev 2>&1 | tail -1; done; done
