# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over smoke() and
# the kernel-level GPU tests; summaries land in gpurun_out/sanitize_*.log.
#   gpurun --timeout 3000 -- 'bash tools/gpu_sanitize.sh'
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SMOKE='import __graft_entry__ as g; g.smoke()'
KTESTS='tests/test_gpu_parity.py -k dw_fwd_bit_exact or dw_bwd_fused or dw_gk or pointwise_fwd_bwd or sgd_bit_exact or toy_step_replay'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 50 \
      python -c "$SMOKE" > gpurun_out/sanitize_${tool}_smoke.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_${tool}_smoke.log
done
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 \
      python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_parity.py \
      -k "dw_fwd_bit_exact or dw_bwd_fused or dw_gk or pointwise_fwd_bwd or sgd_bit_exact or toy_step_replay or prefix_infer or three_layer" \
      > gpurun_out/sanitize_${tool}_kernels.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_${tool}_kernels.log
done
