set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "descriptor or orientation or keypoints_end_to_end or full_size_1920 or rot90 or describe or variants or fed_keypoints or g1_diffusivity_end or 4096x4096" > gpurun_out/gpu_tests_m.log 2>&1
tail -3 gpurun_out/gpu_tests_m.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err
