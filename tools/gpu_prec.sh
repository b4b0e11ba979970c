cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for t in 1 3 4; do PBKD_TF32_TERMS=$t timeout 300 python tools/prec_probe.py; done > gpurun_out/prec.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
