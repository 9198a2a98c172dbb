"""Transaction accounting of an epoch against a clique cache (simulator.py of the reference).

`account_assignment` evaluates the reference's tier rule (simulator.py:132-203) in
the K9 kernel: a neighbour-list read or feature lookup is free on a local hit,
costs NVLink transactions from the lowest-index clique peer holding the vertex,
and PCIe transactions from the CPU otherwise. The same rule decides where the K4
gather fetches each row (cache.FeatureStore), so this report is the transaction
view of what the device path moves. Baseline cache policies and the experiment
CLI are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph, FeatureSpec
from .hardware import CliqueLayout, HardwareSpec
from .planner import CacheAssignment, feature_row_transactions
from .sampling import GpuTrace, SamplingConfig, run_sampling_epoch


@dataclass
class TrafficReport:
    """Per-GPU traffic and hits of one epoch (simulator.py:93-122)."""

    num_gpus: int
    sampling_cpu_txn: np.ndarray
    sampling_peer_txn: np.ndarray
    feature_cpu_txn: np.ndarray
    feature_peer_txn: np.ndarray
    topo_reads: np.ndarray
    topo_local_hits: np.ndarray
    topo_peer_hits: np.ndarray
    feat_lookups: np.ndarray
    feat_local_hits: np.ndarray
    feat_peer_hits: np.ndarray
    traffic_matrix: np.ndarray  # int64 (num_gpus, num_gpus + 1); last column = CPU

    @property
    def topo_hit_rate(self) -> np.ndarray:
        hits = self.topo_local_hits + self.topo_peer_hits
        return np.divide(hits, self.topo_reads, out=np.zeros(self.num_gpus), where=self.topo_reads > 0)

    @property
    def feat_hit_rate(self) -> np.ndarray:
        hits = self.feat_local_hits + self.feat_peer_hits
        return np.divide(hits, self.feat_lookups, out=np.zeros(self.num_gpus), where=self.feat_lookups > 0)

    @property
    def total_cpu_txn(self) -> int:
        return int(self.sampling_cpu_txn.sum() + self.feature_cpu_txn.sum())


_FIELDS = ("topo_reads", "topo_local_hits", "topo_peer_hits", "sampling_cpu_txn", "sampling_peer_txn",
           "feat_lookups", "feat_local_hits", "feat_peer_hits", "feature_cpu_txn", "feature_peer_txn")


def _holders(lists: list[np.ndarray], members: tuple[int, ...], n: int) -> torch.Tensor:
    lib = _lib.lib()
    h = torch.zeros((n + 3) // 4 * 4, dtype=torch.uint8, device="cuda")
    for li, gpu in enumerate(members):
        ids = torch.from_numpy(np.ascontiguousarray(lists[gpu], dtype=np.int64)).cuda()
        _lib.check(lib.gc_mark_holders(ids.data_ptr(), ids.numel(), li, h.data_ptr(), _lib.stream_handle()),
                   "mark_holders")
    return h


def _dev_u64(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()


def account_assignment(traces: list[GpuTrace], assignment: CacheAssignment, layout: CliqueLayout, graph: CsrGraph,
                       spec: HardwareSpec, feat: FeatureSpec) -> TrafficReport:
    """Charge one epoch's access trace against a cache assignment (simulator.py:132-203)."""
    lib = _lib.lib()
    n, G = graph.num_vertices, layout.num_gpus
    rep = {f: np.zeros(G, dtype=np.int64) for f in _FIELDS}
    matrix = np.zeros((G, G + 1), dtype=np.int64)
    row_txns = feature_row_transactions(feat, spec)
    ro = graph.device().c_struct.row_offsets
    for members in layout.cliques:
        k = len(members)
        th = _holders(assignment.topo_vertices, members, n)
        fh = _holders(assignment.feat_vertices, members, n)
        out = torch.zeros(10 + 2 * k, dtype=torch.int64, device="cuda")
        for li, gpu in enumerate(members):
            tr = traces[gpu]
            reads, looks = _dev_u64(tr.topo_reads), _dev_u64(tr.feat_lookups)
            _lib.check(lib.gc_tier_account(ro, n, reads.data_ptr(), looks.data_ptr(), th.data_ptr(), fh.data_ptr(), li,
                                           k, spec.cache_line_bytes, spec.uint32_bytes, row_txns, out.data_ptr(),
                                           _lib.stream_handle()), "tier_account")
            v = out.cpu().numpy()
            for i, f in enumerate(_FIELDS):
                rep[f][gpu] = v[i]
            for lj, src in enumerate(members):
                matrix[gpu, src] += v[10 + lj] + v[10 + k + lj]
            matrix[gpu, G] += v[3] + v[8]
    return TrafficReport(num_gpus=G, traffic_matrix=matrix, **rep)


def simulate_epoch(graph: CsrGraph, seeds_per_gpu, cfg: SamplingConfig, assignment: CacheAssignment,
                   layout: CliqueLayout, spec: HardwareSpec, feat: FeatureSpec, seed: int, epoch: int = 0
                   ) -> TrafficReport:
    """Replay one epoch on the device and count every transaction (simulator.py:206-228)."""
    for lists in (assignment.topo_vertices, assignment.feat_vertices):
        for arr in lists:
            if len(arr) and (arr.min() < 0 or arr.max() >= graph.num_vertices):
                raise ValueError("cache assignment references invalid vertices")
    traces = run_sampling_epoch(graph, seeds_per_gpu, layout, cfg, seed, epoch)
    return account_assignment(traces, assignment, layout, graph, spec, feat)


@dataclass(frozen=True)
class HitRateSummary:
    per_gpu_topo: np.ndarray
    per_gpu_feat: np.ndarray
    aggregate_topo: float
    aggregate_feat: float
    topo_spread: float
    feat_spread: float


def hit_rate_summary(report: TrafficReport) -> HitRateSummary:
    """Per-GPU and aggregate hit rates and the max-min spread (simulator.py:241-256)."""
    topo, feats = report.topo_hit_rate, report.feat_hit_rate
    tr, fl = report.topo_reads.sum(), report.feat_lookups.sum()
    agg_t = float((report.topo_local_hits + report.topo_peer_hits).sum() / tr) if tr else 0.0
    agg_f = float((report.feat_local_hits + report.feat_peer_hits).sum() / fl) if fl else 0.0
    return HitRateSummary(topo, feats, agg_t, agg_f, float(topo.max() - topo.min()) if len(topo) else 0.0,
                          float(feats.max() - feats.min()) if len(feats) else 0.0)
