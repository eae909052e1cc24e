python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
for lev in 1 2; do for sp in 0 1 2 3 4; do echo -n "splits=$sp "; ASB_GEMM_SPLITS=$sp timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1 | sed 's/host enqueue [0-9.]* ms, //'; done; done
for sp in 0 1 2 3 4; do echo -n "splits=$sp "; ASB_GEMM_SPLITS=$sp timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 --prof 2>&1 | tail -2 | head -1; done
