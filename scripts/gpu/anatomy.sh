set -x
timeout 300 python scripts/gemm_timeline.py 8 0.5b 2>&1 | tail -12
timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -3
ASB_DEBUG_SKIP=attn timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -1
ASB_DEBUG_SKIP=qkv,o,gate_up,down timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -1
ASB_DEBUG_SKIP=norm timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -1
timeout 300 python scripts/step_launches.py llama3.1-8b 64 3000 2>&1 | tail -1
