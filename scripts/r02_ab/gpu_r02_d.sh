set -u
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "hessian or keypoints_end_to_end or full_size_1920 or two_pass or descriptors_stage or graph" > gpurun_out/gpu_tests_d.log 2>&1
tail -3 gpurun_out/gpu_tests_d.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
scripts/ncu_full.sh hfused2 k_hess_fused 0
