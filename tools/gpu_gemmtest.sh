cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "0 0" "1 0" "1 1"; do set -- $v
PYTHONPATH=. PBKD_GEMM_TMA=$1 PBKD_PRESPLIT=$2 PBKD_GEMM_PRESPLIT=$2 timeout 120 python tests/gemm_dump.py /tmp/x.npz > gpurun_out/dump_$1$2.log 2>&1; echo "rc=$?" >> gpurun_out/dump_$1$2.log
done
