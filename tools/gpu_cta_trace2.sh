# Per-CTA timelines of the TMA GEMM launches of the eager profiled epoch, from
# the tracer variant (tools/probes/build_variants.sh trace=-DPBKD_GEMM_TRACE_BUILD)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
PBKD_LIB=tools/probes/_build/trace/libpbkd_b200.so PBKD_GEMM_TRACE=1 PBKD_GEMM_TRACE_N=100000 timeout 600 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cta_trace.log 2>&1
echo rc=$?
grep -c "gemm-cta\] launch" gpurun_out/cta_trace.log
python3 tools/cta_trace_summary.py gpurun_out/cta_trace.log ${FIRST:-0} ${COUNT:-400} > gpurun_out/cta_trace_summary.txt
