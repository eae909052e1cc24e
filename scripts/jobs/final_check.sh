timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_full.log 2>&1; tail -3 gpurun_out/gputest_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -m paper_2603_10342_b200.profile_measure --model llama3.2-3b --decode-batch 16 --decode-ctx 3000 --cold 3000 --resume 64 --resume-ctx 3000 --out gpurun_out/b200_profile_llama3.2-3b.json > /dev/null 2> gpurun_out/prof3b.log
cp gpurun_out/b200_profile_llama3.2-3b.json profiles/
timeout 2400 python scripts/policy_compare.py --config c3 --reps 5 --runs mixed_fcfs agentserve agentserve:rbase=4,r0=4 --out gpurun_out/pc_c3_final.json 2>&1 | tail -3 | cut -c1-400
timeout 900 python bench.py > gpurun_out/bench_c3_final.json 2> gpurun_out/bench_c3_final.err; tail -c 600 gpurun_out/bench_c3_final.json
