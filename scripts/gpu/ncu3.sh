timeout 600 python scripts/gemm_bench.py --tokens 64 80 --models llama3.1-8b llama3.2-3b --out gpurun_out/gemm_bench_b64.json 2>&1 | cut -c1-240
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 -c 2500 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>gpurun_out/ncu_launch2.err; tail -2 gpurun_out/ncu_launch2.err
python scripts/ncu_summary.py launches gpurun_out/launches_r1c.csv | head -14
