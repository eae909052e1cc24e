timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for lev in 1 2 4 0; do for v in 0 1; do env $( [ "$v" = 1 ] && echo ASB_NO_POST_NORM=1 ) timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1; done; done
for v in 0 1; do env $( [ "$v" = 1 ] && echo ASB_NO_POST_NORM=1 ) timeout 300 python scripts/step_launches.py llama3.1-8b 64 3000 2>&1 | tail -1; done
