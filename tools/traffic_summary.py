"""DRAM traffic per launch of the TMA GEMM kernel classes from an ncu launch
list (tools/gpu_full.sh: --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum -k regex:umma_t: both TMA GEMM kernels).  Teacher convs are the
launches of the epoch's teacher pass (the first 13 per epoch for VGG-16:
identified by duration > 150 us); the rest are student pointwise GEMMs.
Writes profiles/r1_traffic.json, which bench.py reports as roofline.traffic."""
import collections
import csv
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/traffic.csv"
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/r1_traffic.json"
rows = list(csv.reader(open(path)))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ki, mi, ui, vi = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
ni = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
names = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3}
launch = collections.defaultdict(dict)
for r in rows[h + 1:]:
    launch[int(r[ki])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    if ni is not None:
        names[int(r[ki])] = r[ni]
agg = {"teacher_conv_gemm": [0, 0.0, 0.0], "pointwise_gemm": [0, 0.0, 0.0]}
for _, m in sorted(launch.items()):  # _ = launch id
    dur = m.get("gpu__time_duration.sum", 0.0)
    nm = names.get(_, "")
    if "umma_ts_kernel<3>" in nm or ", 3>" in nm:  # conv kind (implicit im2col) by template argument
        cls = "teacher_conv_gemm"
    elif nm:
        cls = "pointwise_gemm"
    else:  # no kernel names: teacher convs are the long launches
        cls = "teacher_conv_gemm" if dur > 150.0 else "pointwise_gemm"
    a = agg[cls]
    a[0] += 1
    a[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a[2] += dur
res = {k: {"dram_bytes_per_launch": v[1] / v[0], "us_per_launch_serialized": v[2] / v[0], "launches_sampled": v[0],
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (cold-cache, serialised launches)"}
       for k, v in agg.items() if v[0]}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
