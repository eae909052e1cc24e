# Round-end validation on one box: every GPU test, smoke, the reference arm, the default C3 bench line; C5 / C4 AgentServe vs FCFS on the final kernels
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/gputest_full6.log 2>&1; tail -3 gpurun_out/gputest_full6.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke6.txt 2>&1; tail -1 gpurun_out/smoke6.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref6.json 2> gpurun_out/bench_ref6.err; tail -c 300 gpurun_out/bench_ref6.json
timeout 900 python bench.py > gpurun_out/bench_c3_final6.json 2> gpurun_out/bench_c3_final6.err; tail -c 300 gpurun_out/bench_c3_final6.json
timeout 1500 python scripts/policy_compare.py --config c5 --reps 2 --runs mixed_fcfs agentserve --out gpurun_out/pc_c5_final6.json 2>&1 | tail -1 | cut -c1-200
timeout 1500 python scripts/policy_compare.py --config c4 --reps 1 --runs mixed_fcfs agentserve --out gpurun_out/pc_c4_final6.json 2>&1 | tail -1 | cut -c1-200
