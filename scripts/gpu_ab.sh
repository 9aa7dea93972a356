#!/bin/bash
# A/B of library variants / knobs on the headline bench (one GPU, under gpurun):
#   scripts/gpu_ab.sh OUTDIR "cfg1" "cfg2" ...   where cfg = space-separated VAR=value list ("-" = defaults)
# Prints per config: img/s, selected per-kernel ms per step, SM clock.  KAZE_AB_TESTS="expr" first runs the GPU tests
# selected by -k "expr".
set -u
O=$1; shift; mkdir -p $O
if [ -n "${KAZE_AB_TESTS:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$KAZE_AB_TESTS" > $O/tests.log 2>&1; tail -2 $O/tests.log
fi
i=0
for cfg in "$@"; do
  i=$((i+1)); e=""; [ "$cfg" != "-" ] && e="$cfg"
  env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$i.json 2> $O/bench_$i.err
  python - "$O/bench_$i.json" "$cfg" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1])); k = d["kernels"]
    print(sys.argv[2], round(d["value"], 1), {n: round(k[n]["ms_per_step"], 2) for n in ("prefilter", "grad_l1", "cond", "aos_cols", "aos_rows", "hessian", "nms_mark", "describe") if n in k}, d["clocks"]["sm_mhz"])
except Exception as ex:
    print(sys.argv[2], "FAILED", ex)
PY
done
