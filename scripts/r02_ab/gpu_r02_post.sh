#!/bin/bash
# Follow-up checks after the session-3 pass: matcher under compute-sanitizer (racecheck / memcheck / synccheck at
# 4096 x 4096 descriptors: several reference tiles, both column groups' published thresholds), and the pinned-input
# descriptor margin test (writes gpurun_out/describe_margin.json).
set -u
O=gpurun_out/post; mkdir -p $O
for tool in racecheck memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/match_profile.py 4096 > $O/${tool}_match.log 2>&1
  tail -2 $O/${tool}_match.log
done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "pinned_keypoints" > $O/margin_test.log 2>&1; tail -2 $O/margin_test.log
cat gpurun_out/describe_margin.json 2>/dev/null
