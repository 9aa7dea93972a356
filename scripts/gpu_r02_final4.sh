#!/bin/bash
# Round-2 closing measurement pass at HEAD (one B200, under gpurun): full GPU suite, smoke, the headline bench exactly as the driver
# runs it, the FED bench, the reference arm, a 2-rank gloo dry run of the multi-rank bench on the one GPU, the ncu
# launch list + one --set full capture per main kernel, per-config latencies, the stage sweep, the matcher bench
set -u
O=gpurun_out/final4
mkdir -p $O
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1  # warm the box
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $O/gpu_tests.log 2>&1
echo "gpu tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --scheme fed --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_fed.json 2> $O/bench_fed.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-e2e > $O/multigpu_gloo_dryrun.json 2> $O/multigpu_gloo_dryrun.err
bash scripts/profile_round.sh; mkdir -p $O/prof; mv gpurun_out/prof_*.ncu-rep gpurun_out/prof_*.log gpurun_out/launches.csv $O/prof/ 2>/dev/null
timeout 600 python scripts/configs_bench.py --out $O/configs > $O/configs.log 2>&1
timeout 900 python scripts/stage_sweep.py --out $O/stage_sweep > $O/stage_sweep.log 2>&1
timeout 600 python scripts/match_bench.py --out $O/match_bench.json > $O/match.log 2>&1
# the matcher's own ncu capture (65536^2 random unit descriptors, one k_match_topk launch)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_match_topk -s 2 -c 1 \
  -o $O/prof/prof_match python scripts/match_profile.py 65536 > $O/prof/prof_match.log 2>&1
