set -u
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_i.log 2>&1
tail -3 gpurun_out/gpu_tests_i.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
