for n in 1 4 8; do timeout 120 python scripts/c3_probe.py $n 2>&1 | tail -2 | cut -c1-400; done
timeout 120 python scripts/c3_probe.py 4 agentserve tiny 2>&1 | tail -2 | cut -c1-300
