for n in 12 16 24 32; do echo "n=$n"; timeout 100 python scripts/c3_probe.py $n 2>&1 | tail -3 | cut -c1-400; done
