timeout 300 ./scripts/probes/stream_bin 2>&1 | tee gpurun_out/stream_probe.txt
