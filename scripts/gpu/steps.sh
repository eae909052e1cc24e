timeout 600 python scripts/step_launches.py llama3.2-3b 32 3000 2>&1 | tail -1
timeout 600 python scripts/step_launches.py qwen2.5-7b 64 8192 2>&1 | tail -1
timeout 600 python scripts/step_launches.py llama3.1-8b 64 3000 2>&1 | tail -1
timeout 600 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -1
