# Final tree, final default (constant theta_high 0.85 tau): engine GPU tests, smoke, default C3 bench line
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_kv_registry_gpu.py -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke9.txt 2>&1; tail -1 gpurun_out/smoke9.txt
timeout 900 python bench.py > gpurun_out/bench_c3_final9.json 2> gpurun_out/bench_c3_final9.err; tail -c 300 gpurun_out/bench_c3_final9.json
