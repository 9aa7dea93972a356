set -u
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_o.log 2>&1
tail -3 gpurun_out/gpu_tests_o.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $BARGS > gpurun_out/bench_o_$tag.json 2> gpurun_out/bench_o_$tag.err; }
BARGS="" run ov0 KAZE_OVERLAP=0
BARGS="" run ov1 KAZE_OVERLAP=1
BARGS="" run ov1o3 KAZE_OVERLAP=1 KAZE_DESC_OCC=3
BARGS="" run ov1o2 KAZE_OVERLAP=1 KAZE_DESC_OCC=2
BARGS="--batch 32" run ov1b32 KAZE_OVERLAP=1
BARGS="--batch 32" run ov1o3b32 KAZE_OVERLAP=1 KAZE_DESC_OCC=3
