python -m paper_2603_10342_b200.profile_measure --model qwen2.5-7b --decode-batch 32 --decode-ctx 8192 --cold 8192 --resume 256 --resume-ctx 8192 --out gpurun_out/b200_profile_qwen2.5-7b.json > /dev/null 2> gpurun_out/prof7b.log
cp gpurun_out/b200_profile_qwen2.5-7b.json profiles/
python -c "
import json; from paper_2603_10342_b200 import workloads as w
p,m=w.load_profile('qwen2.5-7b'); print(json.dumps(w.calibrate(p,m)))"
timeout 2400 python scripts/policy_compare.py --config c4 --reps 2 --runs mixed_fcfs agentserve agentserve:rbase=2,r0=2 agentserve:rbase=3,r0=3 --out gpurun_out/pc_c4_v3.json 2>&1 | tail -4 | cut -c1-420
