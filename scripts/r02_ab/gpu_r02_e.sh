set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "descriptor or orientation or keypoints_end_to_end or full_size_1920 or graph or rot90 or describe" > gpurun_out/gpu_tests_e.log 2>&1
tail -3 gpurun_out/gpu_tests_e.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
scripts/ncu_full.sh desc2 k_describe 0
