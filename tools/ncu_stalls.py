"""Top SASS lines by warp-stall samples for one kernel of an ncu report.
Usage: python tools/ncu_stalls.py rep.ncu-rep <kernel-regex> [launch-skip] [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
i = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
data, seen = [], set()
for r in rows[2:]:
    if len(r) <= i or r[0] in seen:
        continue
    seen.add(r[0])
    try:
        data.append((float(r[i]), r[0][-5:], r[src].strip()[:80]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
for v, a, s in sorted(data, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  {a}  {s}")
