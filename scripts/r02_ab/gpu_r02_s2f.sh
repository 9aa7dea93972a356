set -u
O=gpurun_out/s2f; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "keypoints_end or full_size_1920" > $O/tests.log 2>&1
tail -2 $O/tests.log
for cfg in "KAZE_NMS_LB=7" "KAZE_NMS_LB=14" "KAZE_NMS_LB=107"; do
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  python -c "import json,sys; d=json.load(open('$O/bench_$cfg.json')); k=d['kernels']; print('$cfg', round(d['value'],1), [ (n, round(k[n]['ms_per_step'],2)) for n in ('nms_mark','hessian')], d['clocks']['sm_mhz'])"
done
