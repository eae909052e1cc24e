T="tests/test_device_vs_hf_gpu.py"
for r in 1 2 3; do echo "== run $r"; timeout 900 python -m pytest -q -x -s "$T" 2>&1 | grep -E "worst|AssertionError: \(|passed|failed" | head -3; done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_full.log 2>&1; tail -3 gpurun_out/gputest_full.log
