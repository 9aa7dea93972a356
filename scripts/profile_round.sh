#!/bin/bash
# One-GPU profiling pass for the round's profiles/ (run under gpurun):
#   launch list of a short bench run (32 images, one launch batch = the bench launch configuration) + one `ncu --set full` capture of each main kernel.
set -u
export KAZE_BENCH_ALLOW_SHORT=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --images 32 --batch 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for kv in cols:k_aos_cols:4 rows:k_aos_rows_cta:4 cond:k_cond2:3 hfused:k_hess_fused:0 \
          nms:k_nms_mark:0 desc:k_describe:0 emit:k_kp_emit:0 pre:k_prefilter:0 khist:k_khist:0 ${KAZE_PROFILE_EXTRA:-}; do
  IFS=: read t r sk <<< "$kv"
  scripts/ncu_full.sh "$t" "$r" "$sk"
done
