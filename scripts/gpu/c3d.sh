timeout 100 python scripts/c3_probe.py 32 2>&1 | tail -3 | cut -c1-600
