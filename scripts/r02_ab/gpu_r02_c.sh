set -u
for kv in desc:k_describe:0 hfused:k_hess_fused:0 cols:k_aos_cols:4 nms:k_nms_mark:0 rows:k_aos_rows_cta:4; do
  IFS=: read t r sk <<< "$kv"
  scripts/ncu_full.sh "$t" "$r" "$sk"
done
