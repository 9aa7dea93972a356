set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "descriptor or orientation or keypoints_end_to_end or full_size_1920 or rot90 or describe or graph or host_path or batch or capacity or memory" > gpurun_out/gpu_tests_n.log 2>&1
tail -3 gpurun_out/gpu_tests_n.log
for m in 0 1; do KAZE_DESC_DYN=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_n$m.json 2> gpurun_out/bench_n$m.err; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --batch 32 > gpurun_out/bench_n32.json 2> gpurun_out/bench_n32.err
