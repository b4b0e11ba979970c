cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -s -C paper_2012_03096_b200 clean && make -s -C paper_2012_03096_b200 -j16 NVEXTRA=-DPBKD_GEMM_TRACE_BUILD || exit 1
for x in ${XFS:-2 1 0}; do
PBKD_DBG_XF=$x PBKD_GEMM_TRACE=1 PBKD_GEMM_TRACE_N=3 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trace3_$x.log 2>&1
echo "== xf $x"; grep "epilogue start" gpurun_out/trace3_$x.log | sed -n 1,3p; grep "gemm-cta\] launch" gpurun_out/trace3_$x.log | head -3
done
