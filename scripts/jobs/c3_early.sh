# Early controller tick (close the interval once k steps already average above theta_high), C3 10 reps
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve agentserve:early=3 agentserve:early=5 agentserve:early=3,thigh=0.9,tlow=0.5 --out gpurun_out/pc_c3_early.json 2>&1 | tail -1 | cut -c1-200
