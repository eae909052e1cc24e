# Round-end validation of the final tree: every GPU test, smoke, default C3 bench line, reference arm
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/gputest_full7.log 2>&1; tail -3 gpurun_out/gputest_full7.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke7.txt 2>&1; tail -1 gpurun_out/smoke7.txt
timeout 900 python bench.py > gpurun_out/bench_c3_final7.json 2> gpurun_out/bench_c3_final7.err; tail -c 300 gpurun_out/bench_c3_final7.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref7.json 2> gpurun_out/bench_ref7.err; tail -c 200 gpurun_out/bench_ref7.json
