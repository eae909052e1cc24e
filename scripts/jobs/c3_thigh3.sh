# C3: theta_high 0.85-0.9 tau x controller interval 25-50 ms (10 reps); ncu launch list of the FCFS bench episode
timeout 3000 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve agentserve:dt=25 agentserve:dt=35 agentserve:thigh=0.85 agentserve:thigh=0.85,dt=25 --out gpurun_out/pc_c3_thigh3.json 2>&1 | tail -1 | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2_ncu_launches_c3_fcfs.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --policy mixed_fcfs --compare none --horizon-ms 1500 > gpurun_out/ncu_fcfs.out 2> gpurun_out/ncu_fcfs.err; echo "ncu rc=$?"
grep -c gpu__time gpurun_out/r2_ncu_launches_c3_fcfs.csv; grep ERROR gpurun_out/r2_ncu_launches_c3_fcfs.csv | head -3
gzip -f gpurun_out/r2_ncu_launches_c3_fcfs.csv
