#!/bin/bash
# A/B timing under gpurun: runs bench.py (device path only) once per environment setting given as arguments,
# e.g. scripts/ab_bench.sh "KAZE_COLS_M=16" "KAZE_COLS_M=20" ""; writes gpurun_out/ab_<i>.json.
set -u
i=0
for envs in "$@"; do
  env $envs python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  python - "$i" "$envs" <<'PY'
import json, sys
i, envs = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"gpurun_out/ab_{i}.json"))
except Exception as e:
    print(i, envs, "FAILED", e); sys.exit(0)
ks = d["kernels"]
print(f"[{i}] {envs or 'default'}: {d['value']:.1f} img/s, {d['ms_per_step']:.1f} ms/step; " +
      ", ".join(f"{k} {v['ms_per_step']:.1f}" for k, v in ks.items() if v['ms_per_step'] > 1.0))
PY
  i=$((i+1))
done
