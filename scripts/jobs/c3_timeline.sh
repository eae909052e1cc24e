nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc scripts/probes/hmma.cu -o /tmp/hmma && /tmp/hmma
for spec in agentserve mixed_fcfs; do echo "=== $spec"; timeout 300 python scripts/episode_timeline.py --config c3 --spec $spec; done
timeout 1200 python -m pytest tests/test_forward_c4c5_gpu.py -x -q -s 2>&1 | grep -E "near-ties|passed|failed|Error" | head -20
