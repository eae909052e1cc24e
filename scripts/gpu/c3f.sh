timeout 120 python scripts/c3_probe.py 32 2>&1 | tail -2 | cut -c1-500
timeout 120 python scripts/c3_probe.py 32 mixed_fcfs 2>&1 | tail -2 | cut -c1-500
timeout 600 python -m pytest tests/test_engine_gpu.py -x -q 2>&1 | tail -1
