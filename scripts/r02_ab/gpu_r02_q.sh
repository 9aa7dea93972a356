set -u
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fed" > gpurun_out/gpu_tests_q.log 2>&1
tail -5 gpurun_out/gpu_tests_q.log
for m in 0 1; do KAZE_FED_REG=$m timeout 600 python bench.py --scheme fed --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_q_fed$m.json 2> gpurun_out/bench_q_fed$m.err; done
KAZE_BENCH_ALLOW_SHORT=1 timeout 600 ncu --set full --clock-control none -k "regex:k_fed" -s 2 -c 1 -o gpurun_out/prof_fedreg python bench.py --scheme fed --images 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_fedreg.log 2>&1
