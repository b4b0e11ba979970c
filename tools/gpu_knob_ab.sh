# A/B of one on/off knob (KNOB=<env var>): bitwise comparison of VGG-16 blocks
# 1-3 results (knob 0 vs default), 2x bench A/B, then the GPU tests (PYTEST_K).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_2012_03096_b200/libpbkd_b200.so; export PYTHONPATH=$GRAFT_REPO_ROOT
env $KNOB=0 timeout 300 python tools/probes/block1_bits.py $L gpurun_out/k0.npz > gpurun_out/bits.log 2>&1
timeout 300 python tools/probes/block1_bits.py $L gpurun_out/k1.npz >> gpurun_out/bits.log 2>&1
python tools/probes/cmp_npz.py gpurun_out/k0.npz gpurun_out/k1.npz >> gpurun_out/bits.log 2>&1
bash tools/gpu_ab_env.sh "$KNOB=0" "$KNOB=1" "$KNOB=0" "$KNOB=1" > gpurun_out/ab.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} -p no:cacheprovider --timeout=600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
