timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_forward_gpu.py -x -q 2>&1 | tail -2
ASB_DEBUG_SKIP=attn timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 2>&1 | tail -1
for sp in 1 2 4 8 16; do echo "max_splits $sp"; ASB_DECODE_MAX_SPLITS=$sp timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 2>&1 | tail -1; done
for w in "2 4" "4 8" "8 8"; do set -- $w; echo "warps $1 stages $2"; ASB_DECODE_WARPS=$1 ASB_DECODE_STAGES=$2 timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 2>&1 | tail -1; done
ASB_ATTN_COMBINE=1 timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 2>&1 | tail -1
for sk in qkv o; do echo "skip $sk"; ASB_DEBUG_SKIP=$sk timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 2>&1 | tail -1; done
