timeout 600 python scripts/episode_stats.py 2>&1 | tail -40
