for lev in 1 0; do timeout 300 python scripts/mk_timeline.py qwen2.5-0.5b 8 2048 --level=$lev 2>&1 | tail -4; done
timeout 300 python scripts/mk_timeline.py tiny 8 500 2>&1 | tail -4
