# Admitted-chunk attention: packed (token, head) columns vs one item per token vs prefill
# attention, decode step time by partition (B rows + a 16-token chunk, ctx 3000), then parity.
set -u
out=gpurun_out/chunk_pack.txt
: > $out
for lv in 3 4 6 0; do
  for mode in 1 2 0; do
    echo "mode=$mode level=$lv" >> $out
    ASB_CHUNK_AS_DECODE=$mode timeout 120 python scripts/step_launches.py llama3.2-3b 6 3000 --chunk=16 --level=$lv --prof >> $out 2>&1
  done
done
timeout 900 python -m pytest -q -x tests/test_forward_gpu.py tests/test_attn_paths_gpu.py tests/test_forward_c4c5_gpu.py tests/test_determinism_gpu.py > gpurun_out/chunk_pack_tests.txt 2>&1
tail -3 gpurun_out/chunk_pack_tests.txt >> $out
