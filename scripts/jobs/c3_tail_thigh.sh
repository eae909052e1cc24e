# C3 TPOT tail anatomy with theta_high = 0.9 tau, then the ncu launch list of the C3 bench
bash scripts/jobs/c3_tail.sh > gpurun_out/c3_tail_thigh.txt 2>&1; grep -E "===|metrics|gaps >= p95" gpurun_out/c3_tail_thigh.txt | cut -c1-300
bash scripts/jobs/ncu_c3_launches.sh
python scripts/ncu_summary.py launches gpurun_out/r2_ncu_launches_c3_bench.csv.gz > gpurun_out/ncu_c3_launch_summary.txt 2>&1; head -30 gpurun_out/ncu_c3_launch_summary.txt
