# C3 TPOT tail anatomy on the final tree and default controller (AgentServe and FCFS)
bash scripts/jobs/c3_tail.sh > gpurun_out/c3_tail_final.txt 2>&1; grep -E "===|metrics|gaps >= p95" gpurun_out/c3_tail_final.txt | cut -c1-300
