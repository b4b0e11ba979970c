# per-chunk time vs persistent grid size (is the GEMM pipeline bandwidth- or latency-bound?)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -s -C paper_2012_03096_b200 clean && make -s -C paper_2012_03096_b200 -j16 NVEXTRA=-DPBKD_GEMM_TRACE_BUILD || exit 1
for g in 148 74 37; do
PBKD_GEMM_GRID_MAX=$g PBKD_GEMM_TRACE=1 PBKD_GEMM_TRACE_N=100000 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/gridcap_$g.log 2>&1
echo "== grid cap $g"; python3 tools/cta_trace_summary.py gpurun_out/gridcap_$g.log 0 26 | cut -c1-170
done
