"""Key metrics of every kernel in an ncu report: time, warp-inst, issue/ALU/FMA pipe,
occupancy, registers and the top warp-stall reasons.

    python tools/ncu_quick.py REPORT.ncu-rep
"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def g(r, k):
    try:
        return float(r[col[k]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


for r in data:
    name = r[col["Kernel Name"]][:60]
    stalls = {h.split("warp_issue_stalled_")[1].split("_per")[0]: g(r, h) for h in hdr
              if h.startswith("smsp__average_warp_latency_issue_stalled_") or
              (h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct"))}
    tot = sum(v for v in stalls.values() if v == v) or 1
    top = sorted(stalls.items(), key=lambda kv: -(kv[1] if kv[1] == kv[1] else 0))[:6]
    print(f"{name}  {g(r, 'gpu__time_duration.sum') / 1e3:.1f} us  inst {g(r, 'smsp__inst_executed.sum'):.4g}  "
          f"issue {g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"alu {g(r, 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"fma {g(r, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"occ {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"regs {g(r, 'launch__registers_per_thread'):.0f}  grid {g(r, 'launch__grid_size'):.0f}")
    print("   stalls:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top))
