# theta_high = 0.9 tau default: C3 bench line, C5 and C4 AgentServe vs FCFS
timeout 900 python bench.py > gpurun_out/bench_c3_thigh.json 2> gpurun_out/bench_c3_thigh.err; tail -c 300 gpurun_out/bench_c3_thigh.json
timeout 1500 python scripts/policy_compare.py --config c5 --reps 2 --runs mixed_fcfs agentserve agentserve:thigh=1.0 --out gpurun_out/pc_c5_thigh.json 2>&1 | tail -1 | cut -c1-200
timeout 1500 python scripts/policy_compare.py --config c4 --reps 1 --runs mixed_fcfs agentserve agentserve:thigh=1.0 --out gpurun_out/pc_c4_thigh.json 2>&1 | tail -1 | cut -c1-200
