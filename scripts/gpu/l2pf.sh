python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -1
for lev in 1 2 4 0; do for pf in 0 8 16 32; do echo -n "pf=$pf "; ASB_GEMM_L2PF=$pf timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1; done; done
for c in "llama3.2-3b 32 3000" "llama3.1-8b 64 3000"; do for pf in 0 8 16; do echo -n "pf=$pf "; ASB_GEMM_L2PF=$pf timeout 300 python scripts/step_launches.py $c 2>&1 | tail -1; done; done
