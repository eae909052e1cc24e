timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 2500 gpurun_out/bench_c3.json
python -m paper_2603_10342_b200.profile_measure --model llama3.1-8b --decode-batch 32 --decode-ctx 3000 --cold 3000 --resume 64 --resume-ctx 3000 --out gpurun_out/b200_profile_llama3.1-8b.json > /dev/null 2> gpurun_out/prof8b.log
cp gpurun_out/b200_profile_llama3.1-8b.json profiles/
python -m paper_2603_10342_b200.profile_measure --model qwen2.5-7b --decode-batch 32 --decode-ctx 8192 --cold 8192 --resume 256 --resume-ctx 8192 --out gpurun_out/b200_profile_qwen2.5-7b.json > /dev/null 2> gpurun_out/prof7b.log
cp gpurun_out/b200_profile_qwen2.5-7b.json profiles/
timeout 1800 python scripts/policy_compare.py --config c4 --reps 2 --runs mixed_fcfs agentserve --out gpurun_out/pc_c4_v2.json 2>&1 | tail -3
