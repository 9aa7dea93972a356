#!/bin/bash
# Round-2 closing check at HEAD (one B200): the full GPU suite, smoke, the headline bench as the driver runs it,
# and the ncu launch list of a 32-image run.
set -u
O=gpurun_out/head; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
export KAZE_BENCH_ALLOW_SHORT=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --images 32 --batch 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
