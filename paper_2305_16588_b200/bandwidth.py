"""Bandwidths measured on the box, and the cost model's time objective.

The reference's objective is the PCIe transaction count N_total = N_T + N_F (Eqs. 4-8,
planner.py:142-169), charging a 64-byte topology transaction and a 64-byte slice of a
feature row alike, with NVLink neglected. On a B200 the two
host-tier access shapes do not cost the same per byte: neighbour-list reads are short
random reads (1 + ceil(4 deg / 64) lines per list) while feature rows are 400-1024-byte
contiguous reads. `north_star` asks for a cost model "fed with bandwidths measured on the
box", so this module

* measures, through the product's own gather kernel (K4), the GB/s of random host-tier
  reads at both access shapes over buffers as large as the host tier really is (the
  host tier's rate falls with table size on this box: profiles/r01_tiers_c3_lanes.md);
* turns a TrafficEstimate into seconds per epoch: sampling_txns * CLS / topology GB/s
  + feature_misses * row_bytes / feature GB/s.

`planner.search_optimal_plan(..., bandwidths=...)` minimises that time instead of
N_total (the reference objective stays the default and stays bit-exact).
"""

from __future__ import annotations

import ctypes
import json
import time
from dataclasses import asdict, dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .graph import FeatureSpec
from .hardware import HardwareSpec


@dataclass(frozen=True)
class MeasuredBandwidths:
    """Sustained GB/s of the host tier at the two access shapes of the cost model."""

    pcie_topology_gbs: float  # random cache-line (64 B) reads of the host CSR
    pcie_feature_gbs: float  # random feature-row reads of the host feature table
    hbm_gbs: float | None = None
    nvlink_gbs: float | None = None
    source: str = ""

    def to_json(self) -> str:
        return json.dumps(asdict(self))

    @classmethod
    def from_json(cls, text: str) -> "MeasuredBandwidths":
        return cls(**json.loads(text))


def random_read_gbs(host_ptr: int, table_bytes: int, read_bytes: int, reads: int = 1 << 20, reps: int = 3,
                    seed: int = 0) -> float:
    """GB/s of `reads` random, `read_bytes`-aligned reads of `read_bytes` each from the
    mapped host buffer at `host_ptr`, through gc_gather (the host-tier path of K4)."""
    from .cache import FeatureStore

    if read_bytes % 16 or read_bytes <= 0:
        raise ValueError("read_bytes must be a positive multiple of 16")
    n = table_bytes // read_bytes
    if n < 1:
        raise ValueError("table smaller than one read")
    dim = read_bytes // 4
    loc = torch.full((n,), -1, dtype=torch.int32, device="cuda")  # every row host-resident
    fs = FeatureStore(FeatureSpec(dim), 0, 1, loc, [None], None)
    fs.c_struct.host_rows = ctypes.c_void_p(host_ptr)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    ids = torch.randint(0, n, (1, reads), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    cnt = torch.tensor([reads], dtype=torch.int32, device="cuda")
    out = torch.empty((1, reads, dim), dtype=torch.float32, device="cuda")
    fs.gather(ids, cnt, out)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fs.gather(ids, cnt, out)
    e1.record()
    torch.cuda.synchronize()
    return reads * read_bytes * reps / (e0.elapsed_time(e1) / 1000.0) / 1e9


def measure_host_tier(topology_ptr: int, topology_bytes: int, feature_ptr: int, feature_bytes: int,
                      feat: FeatureSpec, spec: HardwareSpec, hbm_gbs: float | None = None,
                      nvlink_gbs: float | None = None) -> MeasuredBandwidths:
    """Measure both host-tier access shapes over the real host tables (pinned, mapped)."""
    t0 = time.perf_counter()
    topo = random_read_gbs(topology_ptr, topology_bytes, spec.cache_line_bytes)
    row = feat.row_bytes if feat.row_bytes % 16 == 0 else spec.cache_line_bytes
    feat_gbs = random_read_gbs(feature_ptr, feature_bytes, row)
    src = (f"gc_gather random reads on this box: {spec.cache_line_bytes} B over {topology_bytes / 1e9:.1f} GB, "
           f"{row} B over {feature_bytes / 1e9:.1f} GB ({time.perf_counter() - t0:.1f} s)")
    return MeasuredBandwidths(topo, feat_gbs, hbm_gbs, nvlink_gbs, src)


def estimate_seconds(est, feat: FeatureSpec, spec: HardwareSpec, bw: MeasuredBandwidths) -> float:
    """Host-tier seconds per epoch of one TrafficEstimate (the time objective)."""
    topo_bytes = float(est.sampling_txns) * spec.cache_line_bytes
    feat_bytes = float(est.feature_misses) * feat.row_bytes
    return topo_bytes / (bw.pcie_topology_gbs * 1e9) + feat_bytes / (bw.pcie_feature_gbs * 1e9)


def spearman(a, b) -> float:
    """Spearman rank correlation (average ranks for ties), as tests/helpers.py:70-89."""
    def ranks(x):
        x = np.asarray(x, dtype=np.float64)
        order = np.argsort(x, kind="stable")
        r = np.empty(len(x), dtype=np.float64)
        i = 0
        while i < len(x):
            j = i
            while j + 1 < len(x) and x[order[j + 1]] == x[order[i]]:
                j += 1
            r[order[i : j + 1]] = (i + j) / 2.0
            i = j + 1
        return r

    ra, rb = ranks(a), ranks(b)
    ra -= ra.mean()
    rb -= rb.mean()
    den = np.sqrt((ra * ra).sum() * (rb * rb).sum())
    return float((ra * rb).sum() / den) if den else 0.0


def load(path: Path) -> MeasuredBandwidths | None:
    p = Path(path)
    return MeasuredBandwidths.from_json(p.read_text()) if p.exists() else None
