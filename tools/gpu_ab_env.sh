# A/B: bench under several env settings given as arguments ("VAR=val VAR2=val" per argument)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$i.log 2>&1
  python3 - "$cfg" gpurun_out/ab_$i.log <<'PY'
import json, sys
for l in open(sys.argv[2]):
    if l.startswith("{"):
        d = json.loads(l)
        ak = d["roofline"]["all_kernels"]
        ks = " ".join(f"{k}={v['ms_per_launch']*1e3:.1f}" for k, v in sorted(ak.items(), key=lambda x: -x[1]["share_of_epoch"])[:9])
        print(f"[{sys.argv[1]}] {d['value']:.0f} samples/s {d['ms_per_step']:.2f} ms | {ks}")
PY
  i=$((i+1))
done
