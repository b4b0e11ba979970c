# Round-2 evidence run (one GPU): GPU tests + smoke, bench lines for every
# BASELINE config, the reference arm, the ncu launch list and DRAM traffic of
# the bench command, one `ncu --set full` capture per hot kernel class, the
# knockout attribution and the e2e phases.  Everything lands in gpurun_out/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1; nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
for c in c1 resnet18 resnet34; do
  timeout 900 python bench.py --config $c --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
timeout 900 python bench.py --config resnet50 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_resnet50.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/bench_ref.log
NCCL_DEBUG=INFO timeout 300 python -m pytest tests/test_multigpu.py -m gpu -q -s -p no:cacheprovider -k gpu_list > gpurun_out/nccl_clique.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:umma_t -c 480 --csv --log-file gpurun_out/traffic.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_traffic.log 2>&1
for k in umma_ts_kernel umma_tma_kernel dw_bwd_kernel dw_fwd_kernel dw_gk_kernel bn_bwd_apply_kernel loss_kernel sgd_kernel reduce_kernel bn_stat_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 60 -c 1 -o gpurun_out/full_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$k.log 2>&1
done
bash tools/gpu_knockout.sh > /dev/null 2>&1
bash tools/gpu_cta_trace2.sh > /dev/null 2>&1
PBKD_TRACE=1 timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
ls -la gpurun_out > gpurun_out/ls.txt
