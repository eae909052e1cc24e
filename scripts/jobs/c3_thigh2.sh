# C3 controller threshold confirmation over 10 reps (theta_high / tau, slots per move)
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve agentserve:thigh=0.9 agentserve:thigh=0.9,dr=2 agentserve:thigh=0.95 agentserve:thigh=0.95,dr=2 agentserve:dr=2 --out gpurun_out/pc_c3_thigh2.json 2>&1 | tail -3 | cut -c1-300
