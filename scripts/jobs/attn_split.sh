timeout 1200 python -m pytest tests/test_forward_gpu.py tests/test_attn_paths_gpu.py tests/test_determinism_gpu.py -q -x 2>&1 | tail -2
bash scripts/jobs/prefill_kernels.sh 2>&1 | tail -4
