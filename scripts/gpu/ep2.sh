timeout 600 python scripts/episode_stats.py 2>&1 | grep -E "steps=|metrics|ticks"
timeout 600 python scripts/episode_stats.py --calibrated-slo 2>&1 | grep -E "steps=|metrics|ticks|\(.*\): n="
