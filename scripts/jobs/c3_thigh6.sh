# C3 confirmation on the final kernels: theta_high 0.85 tau with theta_low 0.4 / 0.45 / 0.5 tau (10 reps)
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve:thigh=0.85,tlow=0.4 agentserve:thigh=0.85 agentserve:thigh=0.85,tlow=0.45 agentserve:thigh=0.9,tlow=0.4 --out gpurun_out/pc_c3_thigh6.json 2>&1 | tail -1 | cut -c1-200
