"""Per-launch device times from an ncu --metrics gpu__time_duration.sum CSV log.
Prints the kernels of the last complete step (from the last expand_groups launch) and
their share. Usage: python tools/launch_list.py launches.csv [marker]"""
import csv
import io
import sys

path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "expand_groups"
lines = [l for l in open(path) if not l.startswith("==")]
rows = list(csv.reader(io.StringIO("".join(lines))))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
unit = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
data = []
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    u = r[unit] if unit is not None else "nsecond"
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    v = v * scale.get(u, 1.0)
    data.append((r[ki].split("(")[0].replace("void ", "")[:48], v))
starts = [i for i, (k, _) in enumerate(data) if marker in k]
if len(starts) >= 2:
    seg = data[starts[-2]:starts[-1]]
else:
    seg = data[starts[-1]:] if starts else data
tot = sum(v for _, v in seg)
for k, v in seg:
    print(f"{v:8.1f} us {100 * v / tot:5.1f}%  {k}")
print(f"{tot:8.1f} us total ({len(seg)} launches)")
