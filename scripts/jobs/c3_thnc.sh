# theta_high by phase: the controller's theta_high during cold bursts, backend.theta_high_no_cold_ms (thnc x tau) otherwise; C3 20 episodes
timeout 3000 python scripts/policy_compare.py --config c3 --reps 20 --runs mixed_fcfs agentserve agentserve:thigh=1.0,thnc=0.85 agentserve:thigh=0.9,thnc=0.8 agentserve:thigh=1.0,thnc=0.8 --out gpurun_out/pc_c3_thnc.json 2>&1 | tail -1 | cut -c1-200
