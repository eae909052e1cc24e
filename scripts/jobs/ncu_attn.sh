timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attention --launch-skip 2 --launch-count 1 \
  -o gpurun_out/ncu_pattn_3b python scripts/kernel_bench.py --models llama3.2-3b --no-decode --reps 1 --out /tmp/k.json > gpurun_out/ncu_pattn.log 2>&1
ncu -i gpurun_out/ncu_pattn_3b.ncu-rep --page source --csv > gpurun_out/ncu_pattn_3b_source.csv 2>&1
ncu -i gpurun_out/ncu_pattn_3b.ncu-rep --page raw --csv > gpurun_out/ncu_pattn_3b_raw.csv 2>&1
ls -la gpurun_out/ncu_pattn_3b*
