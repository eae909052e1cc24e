timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=0 --ncu > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/traffic.csv
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
