"""Transaction accounting of an epoch against a clique cache (simulator.py of the reference).

`account_assignment` evaluates the reference's tier rule (simulator.py:132-203) in
the K9 kernel: a neighbour-list read or feature lookup is free on a local hit,
costs NVLink transactions from the lowest-index clique peer holding the vertex,
and PCIe transactions from the CPU otherwise. The same rule decides where the K4
gather fetches each row (cache.FeatureStore), so this report is the transaction
view of what the device path moves. Baseline cache policies and the experiment
CLI are out of scope.

The comparison cache policies of the reference (gnnlab-replicated, quiver-plus,
pagraph-plus next to legion-hierarchical; simulator.py:41-91, :259-402) run through the
same device kernels: presampling (K2/K3/K5), hotness ranking and prefix split (K6/K8
helpers), the plan search for the hierarchical policy (K7) and the epoch replay + tier
accounting (K9). The LDG partition they need for more than one clique or for
pagraph-plus is computed as the reference does (partition_inter_clique with seed
derive_seed(seed, 0x52), simulator.py:273-276; native gc_partition_ldg) unless one
is passed as `partitioning=`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph, FeatureSpec
from .hardware import CliqueLayout, HardwareSpec
import warnings

from .graph import TrainingSet
from .hardware import block_layout
from .partition import Partitioning, assign_tablets, partition_inter_clique, split_intra_clique
from .planner import (
    CacheAssignment,
    build_candidate_orders,
    distribute_prefix,
    feature_row_transactions,
    hotness_descending_order,
    materialize_assignment,
    search_optimal_plan,
)
from .rng import derive_seed
from .sampling import GpuTrace, HotnessMatrices, SamplingConfig, run_presampling, run_sampling_epoch


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


# ---------------------------------------------------------------------------- policies
POLICY_HIERARCHICAL = "legion-hierarchical"
POLICY_REPLICATED = "gnnlab-replicated"
POLICY_QUIVER = "quiver-plus"
POLICY_PAGRAPH = "pagraph-plus"
POLICY_VARIANTS = (POLICY_HIERARCHICAL, POLICY_REPLICATED, POLICY_QUIVER, POLICY_PAGRAPH)
_GLOBAL_SHUFFLE = (POLICY_REPLICATED, POLICY_QUIVER)  # shuffle the training set globally
_NO_NVLINK = (POLICY_REPLICATED, POLICY_PAGRAPH)  # no cache sharing over NVLink


@dataclass(frozen=True)
class CachePolicy:
    """A cache strategy and its per-GPU size (simulator.py:53-84): cache_ratio (fraction
    of |V| feature rows per GPU) or budget_bytes, else the hardware budget / clique size."""

    variant: str
    cache_ratio: float | None = None
    budget_bytes: int | None = None
    delta_alpha: float = 0.01

    def __post_init__(self):
        if self.variant not in POLICY_VARIANTS:
            raise ValueError(f"unknown policy variant {self.variant!r}")
        if self.cache_ratio is not None and self.budget_bytes is not None:
            raise ValueError("give cache_ratio or budget_bytes, not both")

    def per_gpu_bytes(self, graph: CsrGraph, feat: FeatureSpec, spec: HardwareSpec | None = None) -> int:
        if self.cache_ratio is not None:
            return int(round(self.cache_ratio * graph.num_vertices)) * feat.row_bytes
        if self.budget_bytes is not None:
            return self.budget_bytes
        if spec is None:
            raise ValueError("policy has no size parameter and no hardware budget to fall back on")
        return spec.clique_budget_bytes // spec.layout.clique_size

    def per_gpu_rows(self, graph: CsrGraph, feat: FeatureSpec, spec: HardwareSpec) -> int:
        return self.per_gpu_bytes(graph, feat, spec) // feat.row_bytes


def effective_layout(policy: CachePolicy, layout: CliqueLayout) -> CliqueLayout:
    """Baselines that ignore NVLink run with every GPU in its own clique (simulator.py:87-91)."""
    return block_layout(layout.num_gpus, 1) if policy.variant in _NO_NVLINK else layout


def _need_partitioning(partitioning: Partitioning | None, parts: int, graph: CsrGraph, epsilon: float,
                       seed: int) -> Partitioning:
    """The caller's partition, else partition_inter_clique(graph, parts, epsilon,
    derive_seed(seed, 0x52)) as the reference computes it (simulator.py:273, :276)."""
    if partitioning is not None:
        if partitioning.num_parts != parts:
            raise ValueError(f"partitioning has {partitioning.num_parts} parts, this policy needs {parts}")
        return partitioning
    return partition_inter_clique(graph, parts, epsilon, derive_seed(seed, 0x52))


def policy_seed_pools(policy: CachePolicy, graph: CsrGraph, training: TrainingSet, layout: CliqueLayout, seed: int,
                      epsilon: float = 0.05, partitioning: Partitioning | None = None) -> list[np.ndarray]:
    """Per-GPU seed pools under the policy's shuffling discipline (simulator.py:259-278)."""
    num_gpus = layout.num_gpus
    if policy.variant in _GLOBAL_SHUFFLE:
        perm = np.random.default_rng(derive_seed(seed, 0x51)).permutation(training.vertex_ids)
        return [np.sort(perm[g::num_gpus]) for g in range(num_gpus)]
    if policy.variant == POLICY_PAGRAPH:
        parts = _need_partitioning(partitioning, num_gpus, graph, epsilon, seed)
        ids = training.vertex_ids
        return [ids[parts.assignments[ids] == g] for g in range(num_gpus)]
    parts = _need_partitioning(partitioning, layout.clique_count, graph, epsilon, seed)
    return assign_tablets(split_intra_clique(training, parts, layout), layout)


def build_policy_cache(policy: CachePolicy, hotness: list[HotnessMatrices], layout: CliqueLayout, graph: CsrGraph,
                       feat: FeatureSpec, spec: HardwareSpec) -> CacheAssignment:
    """The cache each policy fills from the presampled hotness (simulator.py:281-347):
    gnnlab-replicated, one global hottest-row prefix on every GPU; quiver-plus, a
    clique-size prefix of the global order split by local preference inside each
    clique; pagraph-plus, each GPU's own hottest rows; legion-hierarchical, the plan
    search over each clique's hotness."""
    n = graph.num_vertices
    num_gpus = layout.num_gpus
    rows_per_gpu = policy.per_gpu_rows(graph, feat, spec)
    if policy.variant == POLICY_HIERARCHICAL:
        budget = policy.per_gpu_bytes(graph, feat, spec) * layout.clique_size
        orders, plans = [], []
        for hot in hotness:
            o = build_candidate_orders(hot)
            plan, _ = search_optimal_plan(o, budget, policy.delta_alpha, graph, feat, spec, hot.sampling_txn_total)
            orders.append(o)
            plans.append(plan)
        return materialize_assignment(orders, plans, layout, graph, feat, spec)
    out = CacheAssignment.empty(num_gpus)
    global_feat = np.zeros(n, dtype=np.int64)
    for hot in hotness:
        global_feat += hot.feat_hotness.sum(axis=0)
    global_order = hotness_descending_order(global_feat)
    if policy.variant == POLICY_REPLICATED:
        prefix = global_order[: min(rows_per_gpu, n)]
        for gpu in range(num_gpus):
            out.feat_vertices[gpu] = prefix.copy()
            out.feat_bytes[gpu] = len(prefix) * feat.row_bytes
        return out
    if policy.variant == POLICY_QUIVER:
        if layout.clique_size == 1:
            warnings.warn("quiver-plus with single-GPU cliques degrades to gnnlab-replicated")
        for ci, members in enumerate(layout.cliques):
            k = len(members)
            prefix = global_order[: min(rows_per_gpu * k, n)]
            owner = np.argmax(hotness[ci].feat_hotness, axis=0).astype(np.int32)
            queues = distribute_prefix(prefix, owner, k)
            for li, gpu in enumerate(members):
                q = queues[li]
                out.feat_vertices[gpu] = q
                out.feat_bytes[gpu] = len(q) * feat.row_bytes
        return out
    for ci, members in enumerate(layout.cliques):  # pagraph-plus
        for li, gpu in enumerate(members):
            prefix = hotness_descending_order(hotness[ci].feat_hotness[li])[: min(rows_per_gpu, n)]
            out.feat_vertices[gpu] = prefix
            out.feat_bytes[gpu] = len(prefix) * feat.row_bytes
    return out


@dataclass
class PolicyRun:
    """Everything one policy produced on one configuration (simulator.py:350-359)."""

    policy: CachePolicy
    layout: CliqueLayout
    pools: list
    hotness: list
    assignment: CacheAssignment
    report: TrafficReport


def run_policy_pipeline(policy: CachePolicy, graph: CsrGraph, training: TrainingSet, layout: CliqueLayout,
                        cfg: SamplingConfig, spec: HardwareSpec, feat: FeatureSpec, master_seed: int,
                        epsilon: float = 0.05, partitioning: Partitioning | None = None) -> PolicyRun:
    """Seed pools, presampling, the policy's cache and one fresh simulated epoch
    (simulator.py:362-402), all sampling and accounting on the device."""
    lay = effective_layout(policy, layout)
    spec_eff = HardwareSpec(layout=lay, clique_budget_bytes=policy.per_gpu_bytes(graph, feat, spec) * lay.clique_size,
                            cache_line_bytes=spec.cache_line_bytes, uint32_bytes=spec.uint32_bytes,
                            uint64_bytes=spec.uint64_bytes, float32_bytes=spec.float32_bytes)
    pools = policy_seed_pools(policy, graph, training, lay, master_seed, epsilon, partitioning)
    pcfg = SamplingConfig(fanouts=cfg.fanouts, batch_size=cfg.batch_size, presample_epochs=cfg.presample_epochs,
                          seed=derive_seed(master_seed, 0x10))
    hotness = run_presampling(graph, pools, lay, pcfg, spec_eff)
    assignment = build_policy_cache(policy, hotness, lay, graph, feat, spec_eff)
    report = simulate_epoch(graph, pools, pcfg, assignment, lay, spec_eff, feat, seed=derive_seed(master_seed, 0x20))
    return PolicyRun(policy, lay, pools, hotness, assignment, report)


@dataclass(frozen=True)
class SweepPoint:
    """One GPU count of a policy sweep (simulator.py:405-409)."""

    gpu_count: int
    total_cpu_txn: int
    normalized: float


def sweep_gpus(policy: CachePolicy, gpu_counts: list[int], graph: CsrGraph, training: TrainingSet,
               cfg: SamplingConfig, feat: FeatureSpec, clique_size: int = 2, seed: int = 0, epsilon: float = 0.05,
               cache_line_bytes: int = 64) -> list[SweepPoint]:
    """Total host-tier PCIe transactions of one policy across GPU counts, normalised
    to the smallest count (simulator.py:412-441): each count runs the whole policy
    pipeline on the device with block cliques of min(clique_size, count) GPUs and a
    clique budget of the policy's per-GPU bytes x clique size."""
    counts = sorted(gpu_counts)
    totals = []
    for count in counts:
        size = min(clique_size, count)
        if count % size:
            raise ValueError(f"gpu count {count} incompatible with clique size {size}")
        layout = block_layout(count, size)
        spec = HardwareSpec(layout=layout, clique_budget_bytes=policy.per_gpu_bytes(graph, feat) * size,
                            cache_line_bytes=cache_line_bytes)
        run = run_policy_pipeline(policy, graph, training, layout, cfg, spec, feat, derive_seed(seed, count), epsilon)
        totals.append(run.report.total_cpu_txn)
    anchor = totals[0] if totals and totals[0] else 1
    return [SweepPoint(c, t, t / anchor) for c, t in zip(counts, totals)]


def write_report_csv(report: TrafficReport, path, provenance: str | None = None) -> None:
    """Per-GPU hit rates and transactions as CSV (simulator.py:444-459)."""
    topo, feats = report.topo_hit_rate, report.feat_hit_rate
    lines = [f"# {provenance}\n"] if provenance else []
    lines.append("gpu,topo_hit_rate,feat_hit_rate,sampling_cpu_txn,feature_cpu_txn,feature_peer_txn\n")
    lines += [f"{g},{topo[g]:.6f},{feats[g]:.6f},{report.sampling_cpu_txn[g]},{report.feature_cpu_txn[g]},"
              f"{report.feature_peer_txn[g]}\n" for g in range(report.num_gpus)]
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(lines)


def write_traffic_matrix_csv(report: TrafficReport, path, provenance: str | None = None) -> None:
    """Traffic matrix rows dest_gpu x (from_gpu*, from_cpu) as CSV (simulator.py:462-470)."""
    lines = [f"# {provenance}\n"] if provenance else []
    cols = [f"from_gpu{g}" for g in range(report.num_gpus)] + ["from_cpu"]
    lines.append("dest_gpu," + ",".join(cols) + "\n")
    lines += [f"{g}," + ",".join(str(int(x)) for x in report.traffic_matrix[g]) + "\n" for g in range(report.num_gpus)]
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(lines)
