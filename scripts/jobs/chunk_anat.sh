for c in 0 16; do for L in 3 9; do timeout 300 python scripts/step_launches.py llama3.2-3b 14 3000 --chunk=$c --level=$L --prof 2>&1 | tail -2; done; done
