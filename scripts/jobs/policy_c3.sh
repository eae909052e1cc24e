python -m paper_2603_10342_b200.profile_measure --model llama3.2-3b --decode-batch 16 --decode-ctx 3000 --cold 3000 --resume 64 --resume-ctx 3000 --out gpurun_out/b200_profile_llama3.2-3b.json > /dev/null 2> gpurun_out/prof3b.log
cp gpurun_out/b200_profile_llama3.2-3b.json profiles/
python -c "
import json; from paper_2603_10342_b200 import workloads as w
p,m=w.load_profile('llama3.2-3b'); print(json.dumps(w.calibrate(p,m)))"
timeout 2400 python scripts/policy_compare.py --config c3 --reps 5 --runs mixed_fcfs agentserve agentserve:slack=2.0,rbase=3,r0=3 agentserve:rbase=4,r0=4 --out gpurun_out/pc_c3_v6.json 2>&1 | tail -6
timeout 900 python bench.py > gpurun_out/bench_c3_v6.json 2> gpurun_out/bench_c3_v6.err; tail -c 1500 gpurun_out/bench_c3_v6.json
