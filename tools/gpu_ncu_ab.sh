# A/B of library builds by per-kernel device time: ncu launch list (warm
# cache, no clock control) of a 1-epoch bench run per build.
# usage: tools/gpu_ncu_ab.sh name=path/to/libpbkd_b200.so ...  ("name=" = in-tree build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
K=${NCU_KERNELS:-regex:"umma_tma|dw_|bn_|loss|sgd|reduce|scatter"}
for spec in "$@"; do
  name=${spec%%=*}; lib=${spec#*=}
  PBKD_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k $K \
    --launch-skip ${NCU_SKIP:-0} -c ${NCU_COUNT:-1200} --csv --log-file gpurun_out/ncu_ab_$name.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ab_$name.log 2>&1
  echo "== $name"; python3 tools/launch_summary.py gpurun_out/ncu_ab_$name.csv | head -${NCU_TOP:-16}
done
