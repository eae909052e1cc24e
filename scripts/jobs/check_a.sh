for L in 2 3 4 9; do python scripts/step_launches.py llama3.2-3b 16 3000 --level=$L --prof 2>&1 | tail -2; done > gpurun_out/anat3b_b.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_a.log 2>&1; tail -3 gpurun_out/gputest_a.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; tail -c 3000 gpurun_out/bench_a.json
