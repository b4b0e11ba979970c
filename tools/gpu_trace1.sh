# bench on the product build, then CTA-0 chunk timeline of the first teacher conv (tracer build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/gpu_ab_env.sh "PBKD_X=0"
make -s -C paper_2012_03096_b200 clean && make -s -C paper_2012_03096_b200 -j16 NVEXTRA=-DPBKD_GEMM_TRACE_BUILD || exit 1
PBKD_GEMM_TRACE=1 PBKD_GEMM_TRACE_N=100000 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trace1.log 2>&1
python3 tools/cta_trace_summary.py gpurun_out/trace1.log 0 26 | cut -c1-170
