# Final controller and kernels: C3 AgentServe vs FCFS over 20 episodes; C2 over 5
timeout 3000 python scripts/policy_compare.py --config c3 --reps 20 --runs mixed_fcfs agentserve --out gpurun_out/pc_c3_final20.json 2>&1 | tail -1 | cut -c1-200
timeout 1500 python scripts/policy_compare.py --config c2 --reps 5 --runs mixed_fcfs agentserve --out gpurun_out/pc_c2_final.json 2>&1 | tail -1 | cut -c1-200
