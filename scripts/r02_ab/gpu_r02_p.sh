set -u
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_p.log 2>&1
tail -3 gpurun_out/gpu_tests_p.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $BARGS > gpurun_out/bench_p_$tag.json 2> gpurun_out/bench_p_$tag.err; }
BARGS="" run b32
BARGS="--batch 24" run b24
BARGS="--batch 48" run b48
BARGS="" run b32o4 KAZE_DESC_OCC=4
BARGS="" run b32o2 KAZE_DESC_OCC=2
