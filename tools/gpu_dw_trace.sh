# per-CTA phase summary of the depthwise kernels in the eager profiled epoch (tracer build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -s -C paper_2012_03096_b200 clean && make -s -C paper_2012_03096_b200 -j16 NVEXTRA=-DPBKD_GEMM_TRACE_BUILD || exit 1
for k in dw_fwd dw_bwd dw_gk; do
PBKD_CTA_TRACE=$k timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep cta-trace | tail -12 > gpurun_out/dwtrace_$k.log
done
cat gpurun_out/dwtrace_*.log
