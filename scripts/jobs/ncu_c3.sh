# launch list of the C3 bench episode (ncu gpu__time_duration pass, first 4000 launches) and
# DRAM traffic per decode launch at the C3 shape (16 rows, ctx 3000, full device)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2_ncu_launches_c3_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --compare none > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "step/" --csv --log-file gpurun_out/t_c3.csv \
  python scripts/step_launches.py llama3.2-3b 16 3000 --level=0 --ncu > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/t_c3.csv --config c3 --model llama3.2-3b --rows 16 --ctx 3000 --steps 1
cp profiles/ncu_traffic_c3.json gpurun_out/
gzip -f gpurun_out/r2_ncu_launches_c3_bench.csv
