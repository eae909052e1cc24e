timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 -c 4000 --csv --log-file gpurun_out/r2_ncu_launches_c3_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --compare none > gpurun_out/ncu_bench.out 2> gpurun_out/ncu_bench.err; echo "rc=$?"
tail -5 gpurun_out/ncu_bench.err; tail -c 600 gpurun_out/ncu_bench.out
gzip -f gpurun_out/r2_ncu_launches_c3_bench.csv
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "step/" --csv --log-file gpurun_out/t_c3.csv \
  python scripts/step_launches.py llama3.2-3b 16 3000 --level=0 --ncu > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/t_c3.csv --config c3 --model llama3.2-3b --rows 16 --ctx 3000 --steps 1
cp profiles/ncu_traffic_c3.json gpurun_out/
gzip -f gpurun_out/r2_ncu_launches_c3_bench.csv
