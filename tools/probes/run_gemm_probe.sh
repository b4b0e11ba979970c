# GEMM probe under the product library and each diagnosis variant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B=tools/probes/_build
echo "== product"; timeout 120 $B/gemm_probe 50
for v in "$@"; do echo "== $v"; LD_LIBRARY_PATH=$B/$v timeout 120 $B/gemm_probe 50; done
