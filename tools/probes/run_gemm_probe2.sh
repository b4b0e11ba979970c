cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B=tools/probes/_build
echo "== product ksweep"; timeout 200 $B/gemm_probe 30 ksweep
echo "== lean ksweep"; LD_LIBRARY_PATH=$B/lean timeout 200 $B/gemm_probe 30 ksweep
echo "== trace 16 tiles K512"; PBKD_GEMM_TRACE=3 PBKD_GEMM_TRACE_N=1 LD_LIBRARY_PATH=$B/trace timeout 100 $B/gemm_probe 5 one 512 512 512 0
echo "== trace 16 tiles K512 epi1"; PBKD_GEMM_TRACE=3 PBKD_GEMM_TRACE_N=1 LD_LIBRARY_PATH=$B/trace timeout 100 $B/gemm_probe 5 one 512 512 512 1
echo "== trace 64x2 K64 epi1"; PBKD_GEMM_TRACE=3 PBKD_GEMM_TRACE_N=1 LD_LIBRARY_PATH=$B/trace timeout 100 $B/gemm_probe 5 one 32768 64 64 1
