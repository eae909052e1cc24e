# Decode step: stream-launched vs the same forward captured into a CUDA graph and replayed
# (ASB_GRAPH_PROBE=1; lane event time = device time of the step, capture excluded)
for g in 0 1; do
  for c in "qwen2.5-0.5b 8 2048" "qwen2.5-0.5b 8 2048 --level=1" "qwen2.5-0.5b 2 2048" "llama3.2-3b 16 3000" "llama3.2-3b 16 3000 --level=3"; do
    echo -n "graph=$g "; ASB_GRAPH_PROBE=$g timeout 120 python scripts/step_launches.py $c 2>&1 | tail -1
  done
done
