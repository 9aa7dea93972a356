set -u
# refresh after the matcher changes: full GPU suite, smoke, matcher bench, headline bench
O=gpurun_out/s3; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python scripts/match_bench.py --out $O/match_bench.json > $O/match.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
