set -u
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fed or levels_1920" > gpurun_out/gpu_tests_r.log 2>&1
tail -5 gpurun_out/gpu_tests_r.log
timeout 600 python bench.py --scheme fed --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r_fed.json 2> gpurun_out/bench_r_fed.err
KAZE_BENCH_ALLOW_SHORT=1 timeout 600 ncu --set full --clock-control none -k "regex:k_fed" -s 2 -c 1 -o gpurun_out/prof_fedreg2 python bench.py --scheme fed --images 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_fedreg2.log 2>&1
