set -u
O=gpurun_out/s2d; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "launch_order or levels_1920 or full_size_1920 or overlapped or scale_space" > $O/tests.log 2>&1
tail -3 $O/tests.log
for cfg in "KAZE_ALTERNATE=0" "KAZE_ALTERNATE=1" "KAZE_ALTERNATE=0" "KAZE_ALTERNATE=1"; do
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  python -c "import json,sys; d=json.load(open('$O/bench_$cfg.json')); k=d['kernels']; print('$cfg', round(d['value'],1), [ (n, round(k[n]['ms_per_step'],2)) for n in ('cond','aos_cols','aos_rows','hessian')], d['clocks']['sm_mhz'])"
done
