cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout=280 -k "replay" > gpurun_out/replay_default.log 2>&1
PBKD_GEMM_TMA=0 PBKD_CONV_TMA=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout=280 -k "replay" > gpurun_out/replay_reg.log 2>&1
PBKD_PRESPLIT=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout=280 -k "replay" > gpurun_out/replay_nopre.log 2>&1
