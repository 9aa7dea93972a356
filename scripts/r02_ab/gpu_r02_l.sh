set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "contrast_k or levels_1920 or constant" > gpurun_out/gpu_tests_l.log 2>&1
tail -3 gpurun_out/gpu_tests_l.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err
