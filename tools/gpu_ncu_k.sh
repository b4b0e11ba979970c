cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in dw_fwd_kernel dw_bwd_kernel loss_kernel; do
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$k -s 40 -c 1 -o gpurun_out/full_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$k.log 2>&1
done
