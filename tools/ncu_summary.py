"""Summarise an ncu report: one line per profiled kernel with time, DRAM bytes,
throughput, occupancy and registers. Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
want = {
    "Kernel Name": "kernel",
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_act%",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "launch__occupancy_limit_registers": "occ_lim_regs",
}
idx = {w: hdr.index(w) for w in want if w in hdr}
for r in rows[2:]:
    parts = []
    for w, name in want.items():
        if w not in idx:
            continue
        v = r[idx[w]]
        u = units[idx[w]]
        if name == "kernel":
            v = v.split("(")[0][:40]
        elif u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
            mult = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}[u]
            v = f"{float(v.replace(',', '')) * mult:.1f}MB"
        elif u == "nsecond":
            v = f"{float(v.replace(',', '')) / 1000:.1f}"
        elif u == "usecond":
            v = f"{float(v.replace(',', '')):.1f}"
        parts.append(f"{name}={v}")
    print(" ".join(parts))
