#!/bin/bash
# usage: scripts/ncu_full.sh <tag> <kernel-regex> [skip] — one `ncu --set full` capture of one launch (1 GPU)
tag=$1; re=$2; skip=${3:-2}
export KAZE_BENCH_ALLOW_SHORT=1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$re" -s $skip -c 1 \
  -o gpurun_out/prof_${tag} python bench.py --images 4 --batch 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/prof_${tag}.log 2>&1
echo "ncu $tag rc=$?"
