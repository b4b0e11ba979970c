"""Hot basic blocks of one kernel launch in an ncu report (SASS source page):
runs of instructions with equal execution counts, ranked by issued share."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
launch = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
# one table per launch, each preceded by a "Kernel Name" line
tables = [t for t in out.split('"Kernel Name"') if t.strip()]
r = list(csv.reader(io.StringIO('"Kernel Name"' + tables[launch])))
H = r[1]
rows = [x for x in r[2:] if len(x) >= len(H) - 1]
ie = H.index("Instructions Executed")
ws = H.index("Warp Stall Sampling (All Samples)")
tot = sum(float(x[ie] or 0) for x in rows)
print(r[0][1], "warp instructions", int(tot))
blocks, cur = [], None
for x in rows:
    n = float(x[ie] or 0)
    if cur and cur[1] == n:
        cur[2].append(x[1])
        cur[3] += float(x[ws] or 0)
    else:
        cur = [x[0], n, [x[1]], float(x[ws] or 0)]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[1] * len(b[2]))
for b in blocks[:top]:
    print(f"{b[0]} x{int(b[1])} len {len(b[2])} share {b[1] * len(b[2]) / tot * 100:.1f}% stall {b[3]:.0f}")
    print("    " + " | ".join(s.split(",")[0][:34] for s in b[2][:48]))
