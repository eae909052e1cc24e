timeout 900 python scripts/policy_compare.py --config c3 --reps 1 --out gpurun_out/policy_compare_c3.json 2>&1 | cut -c1-330
