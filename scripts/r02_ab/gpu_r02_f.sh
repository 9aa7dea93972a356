set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "keypoints or hessian or full_size_1920 or two_pass or variants or capacity or graph or rot90 or profile" > gpurun_out/gpu_tests_f.log 2>&1
tail -3 gpurun_out/gpu_tests_f.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
KAZE_NMS_LEAN=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_f0.json 2> gpurun_out/bench_f0.err
scripts/ncu_full.sh nms2 k_nms_mark 0
