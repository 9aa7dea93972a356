#!/bin/bash
# usage: scripts/ncu_full.sh <tag> <kernel-regex> [skip] [extra bench args] — one `ncu --set full` capture of one
# launch (1 GPU) in the bench's launch configuration (32 images of 1920x1200 per launch).
tag=$1; re=$2; skip=${3:-2}; shift 3 2>/dev/null; extra="$*"
export KAZE_BENCH_ALLOW_SHORT=1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$re" -s $skip -c 1 \
  -o gpurun_out/prof_${tag} python bench.py --images 32 --batch 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $extra \
  > gpurun_out/prof_${tag}.log 2>&1
echo "ncu $tag rc=$?"
