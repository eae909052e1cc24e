timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -5
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for v in "" 1; do ASB_NO_DGEMV=$v timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -1; done
for v in "" 1; do ASB_NO_DGEMV=$v timeout 300 python scripts/step_launches.py llama3.2-3b 16 3000 2>&1 | tail -1; done
ASB_DEBUG_SKIP=attn timeout 300 python scripts/step_launches.py qwen2.5-0.5b 8 2048 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:dgemv --launch-skip 300 -c 200 --csv --log-file gpurun_out/dgemv_launches.csv python scripts/ncu_decode.py qwen2.5-0.5b 8 2048 4 > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/dgemv_launches.csv | head -40
