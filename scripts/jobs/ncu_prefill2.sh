m=llama3.2-3b
timeout 600 ncu --set full --clock-control none -k regex:"gemm_tn_kernel" --launch-skip 12 --launch-count 4 -o gpurun_out/ncu_prefill2_$m python scripts/kernel_bench.py --models $m --no-decode --reps 1 --out /tmp/k.json > /dev/null 2>&1
ncu -i gpurun_out/ncu_prefill2_$m.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum > gpurun_out/ncu_prefill2_gemm.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attention --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_pattn2_3b python scripts/kernel_bench.py --models $m --no-decode --reps 1 --out /tmp/k.json > /dev/null 2>&1
ncu -i gpurun_out/ncu_pattn2_3b.ncu-rep --page raw --csv > gpurun_out/ncu_pattn2_raw.csv 2>&1
ncu -i gpurun_out/ncu_pattn2_3b.ncu-rep --page source --csv > gpurun_out/ncu_pattn2_source.csv 2>&1
rm -f gpurun_out/*.ncu-rep
