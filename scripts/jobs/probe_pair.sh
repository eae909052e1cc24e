nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc scripts/probes/tma_pair.cu paper_2603_10342_b200/csrc/tmap.cpp -lcuda -o /tmp/tma_pair && /tmp/tma_pair
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_episode.py --quick 2>&1 | tail -15
