# Per-CTA timeline of every TMA GEMM launch of the eager profiled epoch
# (tracer build, not the product build).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -s -C paper_2012_03096_b200 clean && make -s -C paper_2012_03096_b200 -j16 NVEXTRA=-DPBKD_GEMM_TRACE_BUILD || exit 1
PBKD_GEMM_TRACE=1 PBKD_GEMM_TRACE_N=100000 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cta_trace.log 2>&1
echo rc=$?
grep -c gemm-cta gpurun_out/cta_trace.log
