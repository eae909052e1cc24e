timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for kp in 2 1; do echo "KP=$kp"; ASB_GEMM_KP=$kp timeout 600 python scripts/gemm_bench.py --tokens 8 --levels 1 4 0 --models qwen2.5-0.5b 2>&1 | cut -c1-160; done
for kp in 2 1; do echo "KP=$kp"; ASB_GEMM_KP=$kp timeout 600 python scripts/gemm_bench.py --tokens 64 --models llama3.1-8b 2>&1 | cut -c1-170; done
for lev in 1 2 4 0; do for kp in 2 1; do ASB_GEMM_KP=$kp timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1; done; done
