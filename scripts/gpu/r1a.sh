set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; tail -3 gpurun_out/bench_r1a.err
cat gpurun_out/bench_r1a.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 20000 -c 3000 --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>gpurun_out/ncu_launch.err; tail -3 gpurun_out/ncu_launch.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel --launch-skip 776 -c 4 -o gpurun_out/gemm_decode_c2 python scripts/ncu_decode.py qwen2.5-0.5b 8 2048 2 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel -c 2 -o gpurun_out/dattn_c2 python scripts/ncu_decode.py qwen2.5-0.5b 8 2048 2 > gpurun_out/ncu_full2.log 2>&1; tail -3 gpurun_out/ncu_full2.log
