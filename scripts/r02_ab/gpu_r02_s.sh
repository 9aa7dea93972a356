set -u
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fed or levels_1920" > gpurun_out/gpu_tests_s.log 2>&1
tail -3 gpurun_out/gpu_tests_s.log
timeout 600 python bench.py --scheme fed --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_s_fed.json 2> gpurun_out/bench_s_fed.err
