timeout 400 python scripts/policy_compare.py --config c3 --reps 1 --policies agentserve 2>&1 | tail -5 | cut -c1-400
