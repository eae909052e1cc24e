# Final tree with the phase-dependent theta_high: every GPU test, smoke, C3 20-episode comparison (new default vs constant 0.85 tau), default C3 bench line, C5 / C4
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/gputest_full8.log 2>&1; tail -3 gpurun_out/gputest_full8.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke8.txt 2>&1; tail -1 gpurun_out/smoke8.txt
timeout 900 python bench.py > gpurun_out/bench_c3_final8.json 2> gpurun_out/bench_c3_final8.err; tail -c 300 gpurun_out/bench_c3_final8.json
timeout 3000 python scripts/policy_compare.py --config c3 --reps 20 --runs mixed_fcfs agentserve agentserve:thigh=0.85,thnc=0 --out gpurun_out/pc_c3_thnc2.json 2>&1 | tail -1 | cut -c1-200
timeout 1500 python scripts/policy_compare.py --config c5 --reps 2 --runs mixed_fcfs agentserve --out gpurun_out/pc_c5_final8.json 2>&1 | tail -1 | cut -c1-200
timeout 1500 python scripts/policy_compare.py --config c4 --reps 1 --runs mixed_fcfs agentserve --out gpurun_out/pc_c4_final8.json 2>&1 | tail -1 | cut -c1-200
