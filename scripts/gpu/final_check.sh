python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python scripts/kernel_bench.py --out gpurun_out/kernels_v9.json > /dev/null 2>&1; echo kb=$?
