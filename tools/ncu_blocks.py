import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; ie = hdr.index("Instructions Executed"); ws = hdr.index("Warp Stall Sampling (All Samples)")
data = [(r[0], r[1], float(r[ie] or 0), float(r[ws] or 0)) for r in rows[2:] if len(r) > ie]
tot = sum(d[2] for d in data); totw = sum(d[3] for d in data) or 1
blocks = []; cur = None
for a, s, i, w in data:
    if cur and cur[2] == i:
        cur[3] += 1; cur[4].append(s.strip()[:38]); cur[5] += w
    else:
        cur = [a, s, i, 1, [s.strip()[:38]], w]; blocks.append(cur)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
print("total inst %.4g" % tot)
for b in blocks:
    share = b[2] * b[3] / tot * 100
    if share > thr or b[5] / totw * 100 > thr:
        print(b[0][-5:], f"n={b[3]:3d} exec={b[2]:.3g} inst%={share:5.1f} stall%={b[5]/totw*100:5.1f}", " | ".join(b[4][:5]))
