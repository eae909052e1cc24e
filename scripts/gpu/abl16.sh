for ch in 0 16; do
 timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 --chunk=$ch --prof 2>&1 | tail -2
 for sk in attn qkv o gate_up down norm; do echo "skip $sk"; ASB_DEBUG_SKIP=$sk timeout 300 python scripts/step_launches.py qwen2.5-0.5b 2 2300 --level=1 --chunk=$ch 2>&1 | tail -1; done
done
