set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "host or graph or memory" > gpurun_out/gpu_tests_u.log 2>&1
tail -3 gpurun_out/gpu_tests_u.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
