# ncu --set full of the decode attention and decode GEMMs of one Llama-3.2-3B decode step
# (B=16, ctx 3000) on a 32-SM green-context partition (level 2)
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
  -k regex:decode_attn -c 2 -o gpurun_out/r2_l2_dattn python scripts/step_launches.py llama3.2-3b 16 3000 --level=2 --ncu > gpurun_out/ncu_a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" \
  -k regex:gemm_tn -c 4 -o gpurun_out/r2_l2_gemm python scripts/step_launches.py llama3.2-3b 16 3000 --level=2 --ncu > gpurun_out/ncu_b.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" --csv \
  --log-file gpurun_out/r2_l2_launches.csv python scripts/step_launches.py llama3.2-3b 16 3000 --level=2 --ncu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" --csv \
  --log-file gpurun_out/r2_l9_launches.csv python scripts/step_launches.py llama3.2-3b 16 3000 --level=9 --ncu > /dev/null 2>&1
ls -la gpurun_out
