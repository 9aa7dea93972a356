set -u
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "scale_space or levels or keypoints or full_size or constant or minimum or batch or pitched or host or graph or g1 or weickert or prefilter or conductivity or rot90 or overlapped or aos" > gpurun_out/gpu_tests_v.log 2>&1
tail -3 gpurun_out/gpu_tests_v.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
