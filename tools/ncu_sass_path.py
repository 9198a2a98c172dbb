"""Dynamic SASS path of one kernel from an ncu report: every executed instruction with
its executions per launched warp and its share of warp-stall samples.

    python tools/ncu_sass_path.py REPORT.ncu-rep [min_per_warp]
"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ie, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(r[0], r[1].strip(), float(r[ie] or 0), float(r[ws] or 0)) for r in rows[2:] if len(r) > ie]
warps = data[0][2]  # the first instruction runs once per warp
tot = sum(d[2] for d in data)
totw = sum(d[3] for d in data) or 1
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
print(f"warps {warps:.0f}  warp-inst {tot:.4g}  per warp {tot / warps:.1f}")
base = int(data[0][0], 16)
for a, s, i, w in data:
    if i / warps >= thr or w / totw > 0.002:
        print(f"{int(a, 16) - base:6x} {i / warps:7.2f} {w / totw * 100:5.1f}%  {s}")
