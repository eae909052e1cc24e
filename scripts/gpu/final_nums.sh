python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
mkdir -p gpurun_out
timeout 600 python scripts/kernel_bench.py --out gpurun_out/kernels_v10.json > /dev/null 2>&1; echo kb=$?
for c in "llama3.2-3b 32 3000" "qwen2.5-7b 64 8192" "llama3.1-8b 64 3000" "qwen2.5-0.5b 8 2048"; do
  for r in 1 2; do timeout 300 python scripts/step_launches.py $c 2>&1 | tail -1; done
done
