# Copy / summarise the outputs of tools/gpu_round2_profile.sh (gpurun_out/)
# into the committed evidence files profiles/r2_*.
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
G=$R/gpurun_out
P=$R/profiles
grep '^{' $G/bench.log | tail -1 > $P/r2_bench.json
for c in c1 resnet18 resnet34 resnet50 ref; do grep '^{' $G/bench_$c.log | tail -1 > $P/r2_bench_$c.json; done
cp $G/launches.csv $P/r2_launches_vgg16_1gpu.csv
python3 $R/tools/launch_summary.py $P/r2_launches_vgg16_1gpu.csv > $P/r2_launches_vgg16_1gpu.txt
python3 $R/tools/traffic_summary.py $G/traffic.csv $P/r2_traffic.json > /dev/null
python3 $R/tools/ncu_summary.py $G/full_*.ncu-rep > $P/r2_ncu_full_summary.md 2>&1
cp $G/knockout.txt $P/r2_knockout.txt
cp $G/e2e_probe.log $P/r2_e2e_phases.txt
[ -s $G/cta_trace_summary.txt ] && cp $G/cta_trace_summary.txt $P/r2_cta_trace_summary.txt
grep -E "NCCL INFO" $G/nccl_clique.log | grep -iE "comm 0x|Init COMPLETE|nranks|ncclCommInitAll|version" | head -12 \
  > $P/r2_nccl_clique_world1.txt || true
tail -2 $G/pytest_gpu.log
tail -2 $G/smoke.log
