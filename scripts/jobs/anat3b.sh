# decode-step anatomy of the C3 model on green-context partitions (per-category device time)
for B in 16 32; do for L in 1 2 3 4 9; do timeout 300 python scripts/step_launches.py llama3.2-3b $B 3000 --level=$L --prof 2>&1 | tail -2; done; done
