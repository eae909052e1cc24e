python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -3
timeout 300 python -m pytest tests/test_forward_gpu.py tests/test_engine_gpu.py -x -q 2>&1 | tail -2
for T in 8 64; do
  echo "== bulk T=$T"; ASB_NO_DGEMV=1 timeout 120 python scripts/gemm_timeline.py $T 3b 2>&1 | tail -4 | sed 's/start.*1st-acc/.../'
  echo "== pull T=$T"; ASB_GEMM_PULL_REDUCE=1 ASB_NO_DGEMV=1 timeout 120 python scripts/gemm_timeline.py $T 3b 2>&1 | tail -4 | sed 's/start.*1st-acc/.../'
done
