#!/bin/bash
# Matcher epilogue A/B (sign-bit candidate mask + single-candidate insertion vs the compare/select mask).
set -u
O=gpurun_out/m2; mkdir -p $O
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -k "match" > $O/tests.log 2>&1; tail -2 $O/tests.log
for i in 1 2; do
  for v in "" ${MV:-oldmask}; do
    KAZE_LIB_VARIANT=$v timeout 300 python scripts/match_bench.py --reps 20 --out $O/mb_${v:-new}_$i.json > $O/mb_${v:-new}_$i.log 2>&1
    python -c "import json,sys; d=json.load(open('$O/mb_${v:-new}_$i.json')); print('${v:-new}', round(d['kaze_pair']['ms'],3), round(d['random_65536']['ms'],3), round(d['random_65536']['frac'],3), d['kaze_pair']['exact_fallback_rows'], d['random_65536']['exact_fallback_rows'])"
  done
done
