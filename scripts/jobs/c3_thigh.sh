# C3 controller threshold sweep: theta_high as a fraction of tau, controller step size
timeout 3000 python scripts/policy_compare.py --config c3 --reps 5 --runs mixed_fcfs agentserve agentserve:thigh=0.9 agentserve:thigh=0.8 agentserve:thigh=0.8,tlow=0.4 agentserve:thigh=0.7,tlow=0.4 agentserve:dr=2 --out gpurun_out/pc_c3_thigh.json 2>&1 | tail -12 | cut -c1-600
