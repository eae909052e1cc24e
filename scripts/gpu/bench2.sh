timeout 900 python -m paper_2603_10342_b200.profile_measure --model qwen2.5-0.5b --out profiles/b200_profile_qwen2.5-0.5b.json 2>&1 | tail -3
mkdir -p gpurun_out/profiles_new; cp profiles/b200_profile_qwen2.5-0.5b.json gpurun_out/profiles_new/
timeout 600 python scripts/episode_stats.py 2>&1 | grep -E "steps=|metrics|ticks|\(.*\): n="
timeout 900 python bench.py > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; tail -2 gpurun_out/bench_r1c.err; cat gpurun_out/bench_r1c.json
