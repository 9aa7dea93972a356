set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "4096" > gpurun_out/gpu_tests_4096.log 2>&1
for k in 0 1 2 4 8; do
  KAZE_BUILD_SUB=$k timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_sub_$k.json 2> gpurun_out/ab_sub_$k.err
done
