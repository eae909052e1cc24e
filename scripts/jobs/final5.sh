# Round-end validation on one fresh box: every GPU test, smoke, the reference arm, the default bench line
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/gputest_full5.log 2>&1; tail -3 gpurun_out/gputest_full5.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke5.txt 2>&1; tail -1 gpurun_out/smoke5.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref5.json 2> gpurun_out/bench_ref5.err; tail -c 300 gpurun_out/bench_ref5.json
timeout 900 python bench.py > gpurun_out/bench_c3_final5.json 2> gpurun_out/bench_c3_final5.err; tail -c 300 gpurun_out/bench_c3_final5.json
