timeout 1200 python -m paper_2603_10342_b200.profile_measure --model qwen2.5-7b --cold 8192 --decode-batch 64 --decode-ctx 8192 --resume 256 --resume-ctx 8448 --out profiles/b200_profile_qwen2.5-7b.json 2>&1 | tail -2
mkdir -p gpurun_out/pp; cp profiles/b200_profile_qwen2.5-7b.json gpurun_out/pp/
timeout 1200 python scripts/policy_compare.py --config c4 --reps 1 --policies agentserve mixed_fcfs static_partition:4 --out gpurun_out/policy_compare_c4.json 2>&1 | cut -c1-330
