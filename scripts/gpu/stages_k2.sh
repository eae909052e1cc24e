# A/B of the decode GEMM ring depth (KP=2): 5 stages (206 KB smem) vs fewer (co-residency with
# the next/previous kernel's CTAs under PDL)
for st in 5 3 4; do
  sed -i "s/static constexpr int kStages = KP == 2 ? (BN <= 32 ? [0-9] : [0-9])/static constexpr int kStages = KP == 2 ? (BN <= 32 ? $st : $( [ $st -gt 4 ] && echo 4 || echo $st ))/" paper_2603_10342_b200/csrc/gemm.cu
  grep -o "kStages = KP == 2 ? (BN <= 32 ? [0-9] : [0-9])" paper_2603_10342_b200/csrc/gemm.cu
  python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || { echo build failed; exit 1; }
  for lev in 1 2 0; do timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=$lev 2>&1 | tail -1 | sed 's/host enqueue [0-9.]* ms, //'; done
  timeout 300 python scripts/step_launches.py llama3.2-3b 32 3000 2>&1 | tail -1 | sed 's/host enqueue [0-9.]* ms, //'
done
