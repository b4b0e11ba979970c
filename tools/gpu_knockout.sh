# Critical-path attribution: epoch time with each launch class dropped from the graphs (PBKD_KNOCKOUT)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu_ab_env.sh "PBKD_KNOCKOUT=" "PBKD_KNOCKOUT=gemm_conv" "PBKD_KNOCKOUT=gemm_fwd" "PBKD_KNOCKOUT=gemm_dgrad" "PBKD_KNOCKOUT=gemm_wgrad" \
  "PBKD_KNOCKOUT=DwFwdOp" "PBKD_KNOCKOUT=DwBwdOp" "PBKD_KNOCKOUT=DwGkOp" "PBKD_KNOCKOUT=BnBwdApplyOp" "PBKD_KNOCKOUT=ReduceOp" \
  "PBKD_KNOCKOUT=ScatterOp" "PBKD_KNOCKOUT=LossOp" "PBKD_KNOCKOUT=SgdOp" "PBKD_KNOCKOUT=BnStatOp" "PBKD_KNOCKOUT=BnBwdFinOp" 2>&1 | cut -c1-70 | tee gpurun_out/knockout.txt
