for lev in 1 0; do timeout 300 python scripts/attn_timeline.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -8; done
timeout 300 python scripts/attn_timeline.py qwen2.5-0.5b 8 2300 --level=2 2>&1 | tail -8
