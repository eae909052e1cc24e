# Where the C3 TPOT tail comes from, per policy: step time by decode partition / chunk, gap ladder
for spec in ${SPECS:-agentserve mixed_fcfs}; do echo "=== $spec"; timeout 300 python scripts/episode_timeline.py --config c3 --spec $spec --warm 2 | grep -v "^ *[0-9]* *[0-9.]* *[0-9.]* *[0-9.]* *[0-9.]* *[0-9.-]*$"; done
