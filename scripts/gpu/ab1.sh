timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for lev in 1 2 4 0; do for c in "" 1; do echo "level $lev combine=$c"; env $( [ -n "$c" ] && echo ASB_ATTN_COMBINE=1 ) timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 --level=$lev --prof 2>&1 | tail -2; done; done
