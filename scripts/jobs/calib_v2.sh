# Controller interval and resume budget calibrated from the measured profile (workloads.calibrate)
# vs the reference's constants (delta_t 250 ms, budget 256 / 64), against FCFS, C3 / C4 / C5.
timeout 900 python scripts/policy_compare.py --config c3 --reps 10 --runs mixed_fcfs agentserve agentserve:dt=250,b0=256,bmin=64 --out gpurun_out/pc_c3_calib2.json > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3_calib2.json 2> gpurun_out/bench_c3_calib2.err
timeout 1500 python scripts/policy_compare.py --config c5 --reps 2 --runs mixed_fcfs agentserve agentserve:dt=250,b0=256,bmin=64 --out gpurun_out/pc_c5_calib2.json > /dev/null 2>&1
timeout 2400 python scripts/policy_compare.py --config c4 --reps 2 --runs mixed_fcfs agentserve agentserve:dt=250 --out gpurun_out/pc_c4_calib2.json > /dev/null 2>&1
