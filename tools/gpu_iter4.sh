# tests + bench on the product build, then the per-CTA GEMM trace on a tracer build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=400 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
if [ "$TRACE" = 1 ]; then bash tools/gpu_cta_trace.sh; fi
tail -2 gpurun_out/pytest_gpu.log; grep -o '"value": [0-9.]*, "unit": "samples/s", "n_gpus[^}]*ms_per_step": [0-9.]*' gpurun_out/bench.log | head -1; grep -o '"e2e": {"value": [0-9.]*' gpurun_out/bench.log
