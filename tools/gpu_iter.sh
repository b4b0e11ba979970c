cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/probes/tf32_cvt > gpurun_out/tf32_cvt.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout=250 -x -k "gemm_kernels or pointwise or prefix" > gpurun_out/pytest_gemm.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gemm.log
PBKD_PROFILE=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_vgg.log 2>&1
echo "bench rc=$?" >> gpurun_out/prof_vgg.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_tma_kernel -s 2 -c 1 -o gpurun_out/full_conv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_conv.log 2>&1
