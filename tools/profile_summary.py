"""Summarise ncu outputs into profiles/ (launch list shares + full-capture metrics).

    python tools/profile_summary.py --launches gpurun_out/launches_r01.csv \
        --full gpurun_out/epoch_r01.ncu-rep --tag r01
"""

from __future__ import annotations

import argparse
import csv
import json
import subprocess
from collections import OrderedDict, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
STAGE = {  # kernel -> pipeline stage (bench.py stages_ms)
    "k_hop_expand": "hop_expand", "k_unique": "unique_relabel", "k_relabel": "unique_relabel",
    "k_gather": "gather", "k_perm_": "shuffle", "k_scan_": "shuffle",
}
METRICS = [
    ("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
    ("launch__registers_per_thread", "regs"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"), ("smsp__inst_executed.sum", "warp_inst"),
    ("launch__grid_size", "grid"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
]
STALLS = ["long_scoreboard", "barrier", "wait", "math_pipe_throttle", "not_selected", "selected", "short_scoreboard",
          "dispatch_stall", "lg_throttle", "mio_throttle", "branch_resolving", "no_instructions"]


HOP_FANOUT_SLOTS = {"16": 0, "11": 1, "6": 2}  # C2 fanouts (15, 10, 5) -> network template -> hop


def stage_of(name: str, per_launch: bool = False) -> str:
    if per_launch and "k_hop_expand<" in name:
        slots = name.split("k_hop_expand<")[1].split(">")[0].split(",")[0].strip()
        if slots in HOP_FANOUT_SLOTS:
            return f"hop_expand.h{HOP_FANOUT_SLOTS[slots]}"
    for k, v in STAGE.items():
        if k in name:
            return v
    return "torch/other"


def launches(path: Path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    seq = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", ""))) for r in rows[1:] if len(r) > vi]
    # one epoch = from a k_perm_hist (the shuffle's first kernel) to the next; use the last complete one
    starts = [i for i, (n, _) in enumerate(seq) if "k_perm_hist" in n]
    a, b = starts[-2], starts[-1]
    # the bench's 256 MB L2-flush write runs between timed epochs, outside the timed region
    epoch = [(n, t) for n, t in seq[a:b] if "FillFunctor<unsigned char>" not in n]
    tot = sum(t for _, t in epoch)
    by = OrderedDict()
    for n, t in epoch:
        by.setdefault(n, [0, 0.0])
        by[n][0] += 1
        by[n][1] += t
    stages = defaultdict(float)
    for n, (c, t) in by.items():
        stages[stage_of(n)] += t
    return epoch, by, tot, stages


def full(path: Path):
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m, short in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                u = units[i]
                if isinstance(v, float) and u in ("Mbyte", "Gbyte", "Kbyte", "byte"):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                    u = "byte"
                if isinstance(v, float) and u in ("us", "ms", "ns"):
                    v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3}[u]
                    u = "us"
                d[short] = v
        st = {}
        for name in STALLS:
            m = f"smsp__pcsamp_warps_issue_stalled_{name}"
            if m in hdr and r[hdr.index(m)] not in ("", "n/a"):
                st[name] = float(r[hdr.index(m)].replace(",", ""))
        tot = sum(st.values()) or 1.0
        d["stalls"] = {k: 100 * v / tot for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4]}
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=Path)
    ap.add_argument("--full", type=Path)
    ap.add_argument("--tag", default="r01")
    a = ap.parse_args()
    out = ROOT / "profiles"
    out.mkdir(exist_ok=True)
    lines = []
    if a.launches:
        epoch, by, tot, stages = launches(a.launches)
        lines += [f"# Launch list ({a.tag}): one C2 epoch (235 batches), ncu gpu__time_duration.sum",
                  "", "Cold-cache, serialised per-launch times (compare shares, not absolutes). The bench's",
                  "L2-flush write between epochs (outside the timed region) is left out.", "",
                  f"Epoch total: {tot / 1e3:.1f} us over {len(epoch)} launches", "",
                  "| kernel | launches | us | share |", "|---|---|---|---|"]
        for n, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{n[:90]}` | {c} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
        lines += ["", "| stage | us | share |", "|---|---|---|"]
        for s, t in sorted(stages.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {s} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
        (out / f"{a.tag}_launches.md").write_text("\n".join(lines) + "\n")
    if a.full:
        res = full(a.full)
        md = [f"# ncu --set full ({a.tag}): one C2 epoch's hot kernels", "",
              "Replayed per kernel (cold L2, serialised); `--clock-control none`.", "",
              "| kernel | time us | DRAM read MB | DRAM write MB | regs | occupancy % | issue active % | ALU pipe % | "
              "FMA pipe % | DRAM % | L2 hit % | warp inst | top stalls (% of samples) |",
              "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        traffic = defaultdict(lambda: [0.0, 0])
        pipes = {}
        for d in res:
            md.append(f"| `{d['kernel']}` | {d.get('time', 0):.1f} | {d.get('dram_read', 0) / 1e6:.1f} | "
                      f"{d.get('dram_write', 0) / 1e6:.1f} | {d.get('regs')} | {d.get('occupancy_%', 0):.1f} | "
                      f"{d.get('issue_active_%', 0):.1f} | {d.get('alu_pipe_%', 0):.1f} | {d.get('fma_pipe_%', 0):.1f} | "
                      f"{d.get('dram_%', 0):.1f} | {d.get('l2_hit_%', 0):.1f} | {d.get('warp_inst', 0):.3g} | "
                      + ", ".join(f"{k} {v:.0f}" for k, v in d["stalls"].items()) + " |")
            st = stage_of(d["kernel"], per_launch=True)
            traffic[st][0] += d.get("dram_read", 0) + d.get("dram_write", 0)
            traffic[st][1] += 1
            if st.startswith("hop_expand"):
                pipes[st] = {"issue_active_pct": d.get("issue_active_%"), "alu_pipe_pct": d.get("alu_pipe_%"),
                             "fma_pipe_pct": d.get("fma_pipe_%"), "dram_pct": d.get("dram_%"),
                             "warp_inst": d.get("warp_inst"), "top_stalls_pct": d["stalls"]}
        (out / f"{a.tag}_ncu_full.md").write_text("\n".join(md) + "\n")
        # per-launch DRAM traffic by stage, consumed by bench.py's roofline.traffic
        (out / "ncu_traffic.json").write_text(json.dumps(
            {k: v[0] / v[1] for k, v in traffic.items()} | {"_source": f"profiles/{a.tag}_ncu_full.md",
                                                             "_unit": "bytes per launch", "_pipes": pipes},
            indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
