"""Summarise ncu --set full captures (.ncu-rep) into one markdown table row
per profiled launch: duration, DRAM bytes (traffic), DRAM %, tensor-pipe %,
issue-slot %, occupancy, registers, grid."""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "lts__t_sector_hit_rate.pct": "l2_hit",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = row[i].replace(",", "")
                try:
                    d[name] = float(v) * UNIT.get(units[i], 1)
                except ValueError:
                    d[name] = v
        yield d


print("| kernel | grid | time (us) | DRAM read+write (MB) | DRAM % of peak | tensor pipe % | issue % | warps active % | regs |")
print("|---|---|---|---|---|---|---|---|---|")
for p in sys.argv[1:]:
    for d in rows(p):
        mb = (d.get("dram_rd", 0) + d.get("dram_wr", 0)) / 1e6
        print(f"| {d['kernel']} | {int(d.get('grid', 0))} | {d.get('dur_us', 0):.1f} | {mb:.1f} | {d.get('dram_pct', 0):.1f} | "
              f"{d.get('tensor_pct', 0):.1f} | {d.get('issue_pct', 0):.1f} | {d.get('occ_pct', 0):.1f} | {int(d.get('regs', 0))} |")
