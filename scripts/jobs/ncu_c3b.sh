timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 -c 4000 --csv --log-file gpurun_out/r2_ncu_launches_c3_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --compare none > gpurun_out/ncu_bench.out 2> gpurun_out/ncu_bench.err; echo "rc=$?"
tail -5 gpurun_out/ncu_bench.err; tail -c 600 gpurun_out/ncu_bench.out
gzip -f gpurun_out/r2_ncu_launches_c3_bench.csv
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 1200 gpurun_out/bench_ref.json
