cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
PBKD_TRACE=1 timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
EP=3 PBKD_TRACE=1 timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -s 1600 -c 1100 --csv --log-file gpurun_out/launches_warm.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench_warm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_tma_kernel -s 40 -c 2 -o gpurun_out/full_tma python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_tma.log 2>&1
