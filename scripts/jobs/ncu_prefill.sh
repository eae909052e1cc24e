# tensor-pipe utilisation of the prefill GEMM and attention at the C3-C5 shapes (one launch each)
for m in llama3.2-3b qwen2.5-7b llama3.1-8b; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_tn_kernel|prefill_attention" --launch-skip 12 --launch-count 4 \
    -o gpurun_out/ncu_prefill_$m python scripts/kernel_bench.py --models $m --no-decode --reps 1 --out /tmp/k.json > gpurun_out/ncu_prefill_$m.log 2>&1
  ncu -i gpurun_out/ncu_prefill_$m.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,sm__cycles_active.avg,launch__grid_size > gpurun_out/ncu_prefill_$m.csv 2>&1
done
timeout 600 python scripts/kernel_bench.py --models llama3.2-3b qwen2.5-7b llama3.1-8b --no-decode --out /tmp/k2.json 2>&1 | tail -4
