set -u
O=gpurun_out/s2b; mkdir -p $O
KAZE_PDL=0 CUDA_LAUNCH_BLOCKING=1 timeout 600 compute-sanitizer --tool memcheck python scripts/dbg_hess_tma.py 333 257 > $O/memcheck.log 2>&1; tail -2 $O/memcheck.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "hessian or smoke or keypoints_end or full_size_1920" > $O/tests.log 2>&1
tail -3 $O/tests.log
for cfg in "KAZE_HESS_TMA=0" "KAZE_HESS_TMA_R=12" "KAZE_HESS_TMA_R=8" "KAZE_HESS_TMA_R=16" ${EXTRA_CFGS:-}; do
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  python -c "import json,sys; d=json.load(open('$O/bench_$cfg.json')); print('$cfg', round(d['value'],1), round(d['kernels']['hessian']['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
