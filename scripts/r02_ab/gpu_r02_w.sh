set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "keypoints or hessian or full_size_1920 or capacity or rot90 or variants" > gpurun_out/gpu_tests_w.log 2>&1
tail -3 gpurun_out/gpu_tests_w.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_w.json 2> gpurun_out/bench_w.err
