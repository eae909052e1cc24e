# ncu --set full of the decode GEMM (gate_up, 16 tokens) on a 32-SM green-context partition
ncu --set full --clock-control none --import-source on -k regex:gemm_tn --launch-skip 3 --launch-count 1 \
  -o gpurun_out/ncu_gemm_gu_l2 python scripts/gemm_bench.py --models llama3.2-3b --linears gate_up --tokens 16 --levels 2 --paths 1 --iters 5 > gpurun_out/ncu_gemm.log 2>&1
ncu -i gpurun_out/ncu_gemm_gu_l2.ncu-rep --page details --csv > gpurun_out/ncu_gemm_gu_l2_details.csv 2>&1
