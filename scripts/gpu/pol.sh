timeout 900 python -m pytest tests/test_engine_gpu.py -x -q 2>&1 | tail -2
timeout 900 python -m paper_2603_10342_b200.profile_measure --model llama3.2-3b --out profiles/b200_profile_llama3.2-3b.json 2>&1 | tail -1
mkdir -p gpurun_out/pp; cp profiles/b200_profile_llama3.2-3b.json gpurun_out/pp/
timeout 900 python scripts/policy_compare.py --config c2 --reps 2 --out gpurun_out/policy_compare_c2.json 2>&1 | cut -c1-300
timeout 1200 python scripts/policy_compare.py --config c3 --reps 1 --out gpurun_out/policy_compare_c3.json 2>&1 | cut -c1-300
