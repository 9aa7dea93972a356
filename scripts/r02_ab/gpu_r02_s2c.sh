set -u
O=gpurun_out/s2c; mkdir -p $O
KAZE_PDL=0 CUDA_LAUNCH_BLOCKING=1 timeout 600 compute-sanitizer --tool memcheck python scripts/dbg_hess_tma.py 333 257 > $O/memcheck.log 2>&1; tail -4 $O/memcheck.log
bash scripts/gpu_r02_s2b.sh
