set -u
for kv in cond:k_cond2:3 nms:k_nms_mark:0 cols:k_aos_cols:4 hfused:k_hess_fused:0 desc:k_describe:0; do
  IFS=: read t r sk <<< "$kv"
  scripts/ncu_full.sh "s2e_$t" "$r" "$sk"
done
ls -la gpurun_out/
