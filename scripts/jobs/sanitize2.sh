# NOTE: compute-sanitizer has since been closed on the GPU pool (runs under it left GPUs needing a reset); kept as the record of how r2_compute_sanitizer*.txt were produced
# compute-sanitizer over the packed-chunk decode attention (hd128, G=3 columns spanning tokens) and
# the per-token / persistent variants, plus the quick episodes (tiny model, G=2 chunks)
CS=/usr/local/cuda/bin/compute-sanitizer
K="tests/test_forward_gpu.py::test_forward_matches_oracle[hd128-prompt_lens2-6]"
for tool in memcheck racecheck synccheck; do
  echo "== $tool default"; timeout 900 $CS --tool $tool --print-limit 20 python -m pytest -q -x -p no:cacheprovider "$K" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|Error|Hazard" | head -8
done
echo "== memcheck persistent"; ASB_DECODE_PERSIST=1 timeout 900 $CS --tool memcheck python -m pytest -q -x -p no:cacheprovider "$K" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | head -5
echo "== racecheck persistent"; ASB_DECODE_PERSIST=1 timeout 900 $CS --tool racecheck python -m pytest -q -x -p no:cacheprovider "$K" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY" | head -5
echo "== memcheck combine"; ASB_ATTN_COMBINE=1 ASB_ATTN_NO_CLUSTER=1 timeout 900 $CS --tool memcheck python -m pytest -q -x -p no:cacheprovider "$K" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | head -5
echo "== memcheck episodes"; timeout 1200 $CS --tool memcheck python scripts/sanitize_episode.py --quick 2>&1 | grep -E "episode|ERROR SUMMARY" | head -8
