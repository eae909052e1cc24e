timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve --out gpurun_out/pc_c3_final10.json 2>&1 | tail -2 | cut -c1-420
