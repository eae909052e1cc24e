# C3 confirmation: theta_high 0.85 / interval 35 ms candidates vs FCFS twice (FCFS p95 varies run to run), 10 reps each
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve:thigh=0.85 agentserve:dt=35 agentserve:thigh=0.85,dt=35 mixed_fcfs agentserve --out gpurun_out/pc_c3_thigh4.json 2>&1 | tail -1 | cut -c1-200
# launch list of the C3 kernels outside Green Contexts (ncu cannot prepare kernels launched in a
# Green Context: the AgentServe bench episode fails under ncu): 3000-token prefill + B=16 ctx 3000 decode steps, full device
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_ncu_launches_c3_kernels.csv \
  python scripts/kernel_bench.py --models llama3.2-3b --prefill 3000 --decode 16x3000 --reps 1 --out gpurun_out/k_ncu.json > gpurun_out/ncu_k.out 2>&1; echo "ncu rc=$?"
grep -c gpu__time gpurun_out/r2_ncu_launches_c3_kernels.csv; gzip -f gpurun_out/r2_ncu_launches_c3_kernels.csv
