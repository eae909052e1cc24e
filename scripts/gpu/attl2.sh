timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_engine_gpu.py -x -q 2>&1 | tail -2
for lev in 1 0; do timeout 300 python scripts/attn_timeline.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -7; done
for lev in 1 2 4 0; do for c in 0 1; do env $( [ "$c" = 1 ] && echo ASB_ATTN_NO_CLUSTER=1 ) timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1; done; done
