# C3 on the final decode kernels: theta_high 0.75-0.85 tau, theta_low, interval (10 reps)
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve:thigh=0.8 agentserve:thigh=0.75 agentserve:thigh=0.85,tlow=0.4 agentserve:thigh=0.85,dt=50 agentserve:thigh=0.8,dt=50 --out gpurun_out/pc_c3_thigh5.json 2>&1 | tail -1 | cut -c1-200
