cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in dw_fwd_kernel dw_bwd_kernel dw_gk_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 2 -o gpurun_out/full_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
