set -u
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "hessian or keypoints or full_size_1920 or rot90 or variants or descriptors_stage or edge_level or minimum or constant" > gpurun_out/gpu_tests_z.log 2>&1
tail -3 gpurun_out/gpu_tests_z.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_z.json 2> gpurun_out/bench_z.err
