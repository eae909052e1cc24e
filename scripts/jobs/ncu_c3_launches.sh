# launch list of the C3 bench episodes (ncu gpu__time_duration pass): episodes cut at 1.5 s of engine
# time (the cold burst + decode/resume mix) so the whole command finishes under ncu
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2_ncu_launches_c3_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --compare none --horizon-ms 1500 > gpurun_out/ncu_bench.out 2> gpurun_out/ncu_bench.err; echo "rc=$?"
tail -3 gpurun_out/ncu_bench.err; tail -c 300 gpurun_out/ncu_bench.out
gzip -f gpurun_out/r2_ncu_launches_c3_bench.csv
