set -u
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/match_launches.csv python scripts/match_profile.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_match_topk" -s 2 -c 1 -o gpurun_out/prof_match python scripts/match_profile.py > gpurun_out/prof_match.log 2>&1
