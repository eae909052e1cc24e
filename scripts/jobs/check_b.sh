for i in 1 2; do timeout 600 python -m pytest tests/test_device_vs_hf_gpu.py -q -s -k "0.5b" 2>&1 | grep -E "worst|passed|failed|Error"; done > gpurun_out/hf_rerun.log
ASB_DECODE_SPLITS=8 timeout 600 python -m pytest tests/test_device_vs_hf_gpu.py -q -s -k "0.5b" 2>&1 | grep -E "worst|passed|failed|Error" >> gpurun_out/hf_rerun.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_b.log 2>&1; tail -5 gpurun_out/gputest_b.log
