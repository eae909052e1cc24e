for lev in 1 2 0; do for v in 0 1; do ASB_NO_DGEMV=$v timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 --level=$lev --prof 2>&1 | tail -2; done; done
