set -u
KAZE_NMS_LEAN=2 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "keypoints or hessian or full_size_1920 or two_pass or capacity or graph or rot90 or match" > gpurun_out/gpu_tests_g.log 2>&1
tail -3 gpurun_out/gpu_tests_g.log
for m in 1 2; do KAZE_NMS_LEAN=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_g$m.json 2> gpurun_out/bench_g$m.err; done
KAZE_NMS_LEAN=2 scripts/ncu_full.sh nms3 k_nms_mark 0
