timeout 1500 python -m pytest tests/test_forward_c4c5_gpu.py tests/test_forward_gpu.py tests/test_determinism_gpu.py -q -x 2>&1 | tail -2
ASB_TGEMV=1 timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_engine_gpu.py -q -x 2>&1 | tail -2
for L in 3 4; do timeout 300 python scripts/step_launches.py llama3.2-3b 14 3000 --chunk=16 --level=$L 2>&1 | tail -1; done
