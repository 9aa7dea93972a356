set -u
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_t.log 2>&1
tail -3 gpurun_out/gpu_tests_t.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
bash scripts/gpu_r02_ncu32.sh
