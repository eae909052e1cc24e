mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel --launch-skip 600 -c 5 -o gpurun_out/gemm32k2_c2 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 > gpurun_out/ncu_g32.log 2>&1; echo rc=$?; tail -3 gpurun_out/ncu_g32.log
ls -la gpurun_out/*.ncu-rep
