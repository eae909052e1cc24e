timeout 2400 python scripts/policy_compare.py --config c3 --reps 5 --runs mixed_fcfs agentserve agentserve:slack=1.75,rbase=3,r0=3 agentserve:slack=2.0,rbase=3,r0=3 agentserve:slack=2.0 --out gpurun_out/pc_c3_v5.json 2>&1 | tail -6
bash scripts/jobs/ncu_prefill.sh
