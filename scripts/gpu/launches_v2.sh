mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
timeout 1700 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 -c 2500 --csv --log-file gpurun_out/launches_v2.csv python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>gpurun_out/ncu_launch_v2.err; echo rc=$?; tail -1 gpurun_out/ncu_launch_v2.err
gzip -kf gpurun_out/launches_v2.csv
