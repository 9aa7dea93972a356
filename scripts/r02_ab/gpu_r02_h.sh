set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "scale_space or levels or keypoints or full_size_1920 or constant or minimum or batch or pitched or host_path or graph or g1 or weickert or prefilter or conductivity or rot90" > gpurun_out/gpu_tests_h.log 2>&1
tail -3 gpurun_out/gpu_tests_h.log
for m in 0 1; do KAZE_COLS_TMA=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_h$m.json 2> gpurun_out/bench_h$m.err; done
scripts/ncu_full.sh cols2 k_aos_cols 4
