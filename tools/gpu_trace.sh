cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
PBKD_PROFILE=1 PBKD_GEMM_TRACE=120 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/gemm_trace.log 2>&1
