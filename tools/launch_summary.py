"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections, csv, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
limit = int(sys.argv[2]) if len(sys.argv) > 2 else 10**9
rows = list(csv.reader(open(path)))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[h], rows[h + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in data[:limit]:
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1)
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"launches {min(limit, len(data))}, total {tot/1e6:.3f} ms (serialized, cold-cache)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:55s} {c:5d} {t/1e6:9.3f} ms {100*t/tot:5.1f}%  avg {t/c/1e3:8.1f} us")
