cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c1 resnet18 resnet34; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
echo "rc=$?" >> gpurun_out/bench_$c.log
done
