cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B=tools/probes/_build
echo "== product"; timeout 200 $B/gemm_probe 30
echo "== product ksweep"; timeout 200 $B/gemm_probe 30 ksweep
echo "== lean"; LD_LIBRARY_PATH=$B/lean timeout 200 $B/gemm_probe 30
