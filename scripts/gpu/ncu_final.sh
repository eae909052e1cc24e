mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn_kernel --launch-skip 28 -c 2 -o gpurun_out/dattn_c3_final python scripts/ncu_decode.py llama3.2-3b 32 3000 2 > gpurun_out/ncu_da3.log 2>&1; echo da=$?
ls -la gpurun_out/*final*.ncu-rep
