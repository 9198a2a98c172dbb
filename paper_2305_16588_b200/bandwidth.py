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
                    seed: int = 0, sorted_chunk: int = 0) -> float:
    """GB/s of `reads` random, `read_bytes`-aligned reads of `read_bytes` each from the
    mapped host buffer at `host_ptr`, through gc_gather (the host-tier path of K4).
    sorted_chunk > 0 issues the ids in ascending order within each run of that many."""
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
    if sorted_chunk > 0:
        k = -(-reads // sorted_chunk) * sorted_chunk
        pad = torch.full((1, k), torch.iinfo(torch.int32).max, dtype=torch.int32, device="cuda")
        pad[:, :reads] = ids
        ids = pad.view(-1, sorted_chunk).sort(dim=1).values.view(1, -1)[:, :reads].contiguous()
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


def topology_line_gbs(graph, seeds: np.ndarray, fanouts, batch_size: int, stream_key: int = 1, reps: int = 3
                      ) -> tuple[float, dict]:
    """Effective GB/s of host-tier topology reads *inside the sampler* (K2), in the cost
    model's unit of 64-byte lines: the same window of batches is sampled with every
    neighbour list on the host tier (UVA over PCIe) and with the same lists in HBM;
    the extra time divided by the host run's t(v) line count prices one line.
    (Random-read probes of 64-byte lines underestimate this by ~3x on a B200: the
    hop kernel overlaps its row reads with selection work and other CTAs.)"""
    from .cache import TopologyStore
    from .rng import KeyedRng
    from .sampling import WindowSampler, batch_hop_keys

    B = int(batch_size)
    nb = max(1, len(seeds) // B)
    seeds = np.asarray(seeds[: nb * B], dtype=np.int64)
    keys = batch_hop_keys(KeyedRng(stream_key), 0, nb, len(fanouts))
    counts = np.full(nb, B, dtype=np.int32)
    flat = torch.from_numpy(seeds.astype(np.uint32).view(np.int32)).cuda()
    empty = [np.empty(0, dtype=np.int64)]
    times, txn = {}, 0
    for where in ("host", "hbm"):
        ts = TopologyStore(graph, empty, 0, host_full=(where == "host"))
        sp = WindowSampler(graph, fanouts, B, nb, relabel=False, topology=ts)
        sp.load(flat, counts, keys)
        sp.expand()  # warm-up
        torch.cuda.synchronize()
        ts.reset_counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            sp.expand()
        e1.record()
        torch.cuda.synchronize()
        times[where] = e0.elapsed_time(e1) / 1000.0 / reps
        if where == "host":
            txn = ts.tier_counts()["host_txn"] / reps
        sp.bitmap.zero_()
        del sp, ts
    extra = max(times["host"] - times["hbm"], 1e-9)
    gbs = txn * 64 / extra / 1e9
    return gbs, {"batches": nb, "host_s": times["host"], "hbm_s": times["hbm"], "host_lines": txn}


def calibrate_host_tier(graph, seeds: np.ndarray, fanouts, batch_size: int, feature_ptr: int, feature_bytes: int,
                        feat: FeatureSpec, spec: HardwareSpec, hbm_gbs: float | None = None,
                        nvlink_gbs: float | None = None) -> MeasuredBandwidths:
    """Both host-tier costs measured through the product kernels: topology lines by the
    sampler differential (topology_line_gbs), feature rows by the K4 gather of random
    rows over the real host table (the gather is PCIe-bound: its time is the row cost)."""
    t0 = time.perf_counter()
    topo, info = topology_line_gbs(graph, seeds, fanouts, batch_size)
    row = feat.row_bytes if feat.row_bytes % 16 == 0 else spec.cache_line_bytes
    feat_gbs = random_read_gbs(feature_ptr, feature_bytes, row)
    src = (f"sampler differential (host vs HBM topology, {info['batches']} batches, "
           f"{info['host_lines']:.0f} host lines, {info['host_s'] * 1e3:.2f} vs {info['hbm_s'] * 1e3:.2f} ms) and "
           f"K4 random {row} B rows over {feature_bytes / 1e9:.1f} GB ({time.perf_counter() - t0:.1f} s)")
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
