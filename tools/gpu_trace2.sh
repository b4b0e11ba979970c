cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -s -C paper_2012_03096_b200 clean && make -s -C paper_2012_03096_b200 -j16 NVEXTRA=-DPBKD_GEMM_TRACE_BUILD || exit 1
PBKD_GEMM_TRACE=1 PBKD_GEMM_TRACE_N=100000 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trace2.log 2>&1
awk '/\[gemm-trace\] launch 1 BN=128/,/launch 2 BN=128/' gpurun_out/trace2.log | grep "epilogue start" | head -8
awk '/\[gemm-trace\] launch 7 BN=128/,/launch 8 BN=128/' gpurun_out/trace2.log | grep "epilogue start" | head -4
awk '/\[gemm-trace\] launch 13 BN=128/,/launch 14 BN=128/' gpurun_out/trace2.log | grep "epilogue start" | head -4
