T="tests/test_device_vs_hf_gpu.py::test_device_matches_transformers_at_config_lengths[llama3.2-3b-lens1]"
for env in "X=0" "X=1" "X=2" "ASB_DECODE_SPLITS=1" "ASB_DECODE_SPLITS=1 Y=1" "ASB_NO_TGEMV=1 ASB_ATTN_NO_CLUSTER=1"; do
  echo "== $env"; env $env timeout 600 python -m pytest -q -x -s "$T" 2>&1 | grep -E "worst|AssertionError: \(|passed|failed" | head -2
done
