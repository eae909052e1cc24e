python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
for T in 32; do
  echo "== bulk T=$T"; ASB_NO_DGEMV=1 timeout 120 python scripts/gemm_timeline.py $T 3b 2>&1 | tail -4 | sed 's/start.*1st-acc/.../'
  echo "== pull T=$T"; ASB_GEMM_PULL_REDUCE=1 ASB_NO_DGEMV=1 timeout 120 python scripts/gemm_timeline.py $T 3b 2>&1 | tail -4 | sed 's/start.*1st-acc/.../'
done
for c in "llama3.2-3b 32 3000" "qwen2.5-7b 64 8192" "llama3.1-8b 64 3000" "llama3.2-3b 16 3000"; do
  for v in "" 1; do echo "pull=$v $c"; env $( [ -n "$v" ] && echo ASB_GEMM_PULL_REDUCE=1 ) timeout 300 python scripts/step_launches.py $c 2>&1 | tail -1; done
done
