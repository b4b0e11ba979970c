cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B=tools/probes/_build
echo "== product merged"; timeout 200 $B/gemm_probe 30 ksweep 2>&1 | grep -v "^    back" 
echo "== product unmerged (BN64 S=4)"; PBKD_GEMM_MERGE=0 timeout 200 $B/gemm_probe 30 ksweep 2>&1 | grep "N64"
echo "== S=2"; LD_LIBRARY_PATH=$B/s2 timeout 200 $B/gemm_probe 30 ksweep 2>&1 | grep -v "^    back"
