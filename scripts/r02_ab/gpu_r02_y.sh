set -u
for r in 16 12 20; do KAZE_HESS_R=$r timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_y$r.json 2> gpurun_out/bench_y$r.err; done
KAZE_HESS_R=12 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "hessian" > gpurun_out/gpu_tests_y.log 2>&1
tail -2 gpurun_out/gpu_tests_y.log
