nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err; cat gpurun_out/bench_final.json | cut -c1-1500
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 2>&1 | tail -1 | cut -c1-400
timeout 1700 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 -c 2500 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>gpurun_out/ncu_launch_final.err; tail -1 gpurun_out/ncu_launch_final.err
