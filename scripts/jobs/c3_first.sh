set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2603_10342_b200.profile_measure --model llama3.2-3b --decode-batch 16 --decode-ctx 3000 --cold 3000 --resume 64 --resume-ctx 3000 --out gpurun_out/b200_profile_llama3.2-3b.json > /dev/null 2> gpurun_out/prof3b.log
cp gpurun_out/b200_profile_llama3.2-3b.json profiles/
timeout 900 python scripts/policy_compare.py --config c3 --reps 2 --runs mixed_fcfs agentserve agentserve:lend=0 agentserve:calib=0,lend=0 agentserve:slack=2.0 --out gpurun_out/pc_c3_a.json > gpurun_out/pc_c3_a.log 2>&1
timeout 600 python -m pytest tests/test_kv_registry_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
