# Two slots per controller move with the final thresholds (faster climb after the cold burst), C3 20 episodes
timeout 3000 python scripts/policy_compare.py --config c3 --reps 20 --runs mixed_fcfs agentserve agentserve:dr=2 --out gpurun_out/pc_c3_dr2.json 2>&1 | tail -1 | cut -c1-200
