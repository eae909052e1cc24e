python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || exit 1
mkdir -p gpurun_out
for v in 1 0; do
ASB_PREFILL_UNITS=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:prefill --launch-skip 48 -c 6 --csv python scripts/kernel_bench.py --models qwen2.5-0.5b --reps 1 --out /tmp/kb.json 2>/dev/null | grep -E "prefill" | awk -F'","' '{print $5, $7, $8, $NF}' | head -8
done
