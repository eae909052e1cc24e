timeout 1200 python -m pytest tests/test_forward_gpu.py tests/test_attn_paths_gpu.py tests/test_engine_gpu.py tests/test_forward_c4c5_gpu.py -x -q 2>&1 | grep -E "^E|passed|failed" | head -5
for v in 1 0; do echo "== chunk as decode $v"; ASB_CHUNK_AS_DECODE=$v timeout 300 python scripts/step_launches.py llama3.2-3b 14 3000 --chunk=16 2>&1 | tail -1; ASB_CHUNK_AS_DECODE=$v timeout 300 python scripts/step_launches.py llama3.2-3b 14 3000 --chunk=16 --level=4 2>&1 | tail -1; done
timeout 300 python scripts/step_launches.py llama3.2-3b 14 3000 2>&1 | tail -1
for spec in agentserve; do echo "=== $spec"; timeout 300 python scripts/episode_timeline.py --config c3 --spec $spec | tail -14; done
