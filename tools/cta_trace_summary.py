"""Summarise gpurun_out/cta_trace.log (tools/gpu_cta_trace.sh): per TMA GEMM
launch, the in-kernel span, the busiest CTA and a least-squares fit of CTA
duration ~ a + b*chunks + t*tiles."""
import re
import sys

import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cta_trace.log"
first = int(sys.argv[2]) if len(sys.argv) > 2 else 12
count = int(sys.argv[3]) if len(sys.argv) > 3 else 24
launches, cur = [], None
for line in open(path):
    m = re.match(r"\[gemm-cta\] launch (\d+) BN=(\d+) PS=(\d) grid=(\d+) span ([\d.]+)", line)
    if m:
        cur = {"n": int(m[1]), "bn": int(m[2]), "grid": int(m[4]), "span": float(m[5]), "ops": [], "ctas": []}
        launches.append(cur)
        continue
    m = re.match(r"\[gemm-cta\]   op M=(\d+) N=(\d+) K=(\d+) ksplit=(\d+) tiles=(\d+)x(\d+) epi=(\d) conv=(\d)", line)
    if m and cur:
        cur["ops"].append(tuple(int(x) for x in m.groups()))
        continue
    m = re.match(r"\[gemm-cta\]   cta +(\d+) start +([\d.]+) end +([\d.]+) chunks +(\d+) tiles (\d+)", line)
    if m and cur:
        cur["ctas"].append((float(m[2]), float(m[3]), int(m[4]), int(m[5])))
for la in launches[first:first + count]:
    c = np.array(la["ctas"])
    dur = c[:, 1] - c[:, 0]
    i = int(np.argmax(c[:, 1]))
    A = np.c_[np.ones(len(c)), c[:, 2], c[:, 3]]
    a, b, t = np.linalg.lstsq(A, dur, rcond=None)[0]
    epi = sorted({o[6] for o in la["ops"]})
    print(f"#{la['n']:4d} BN={la['bn']:3d} grid={la['grid']:3d} span {la['span']:6.1f} us  end med {np.median(c[:, 1]):6.1f}"
          f"  busiest: {int(c[i, 2]):3d} chunks {int(c[i, 3])} tiles  fit a={a:5.2f} b={b:5.3f}/chunk t={t:5.2f}/tile"
          f"  epi={epi} ops={len(la['ops'])} {[o[:4] for o in la['ops']][:3]}")
