cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout=250 -x -k "gemm_kernels or pointwise or prefix" > gpurun_out/pytest_gemm.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gemm.log
for m in 0 1 2 4 8 7 15; do PBKD_GEMM_DBG=$m timeout 120 python tools/gemm_dbg.py; done > gpurun_out/gemm_dbg.log 2>&1
PBKD_PROFILE=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_vgg.log 2>&1
