"""Cache-candidate ranking, PCIe cost model and plan search (planner.py of the reference).

The O(n) work — clique-wide hotness totals and first-argmax owners, the CSLP ranking
sort, byte/hotness prefix scans, the batched boundary searches for the alpha grid,
and the per-owner split of the cached prefixes — runs in the K6/K7 kernels of
libgnncache_b200.so. The 101-point `_estimate_at` evaluation stays on the host,
where Python's correctly rounded int/int division reproduces the reference exactly
(planner.py:152-169).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph, FeatureSpec
from .hardware import CliqueLayout, HardwareSpec
from .sampling import HotnessMatrices


def _dev_i64(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()


def _temp(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device="cuda")


def device_descending_order(totals: torch.Tensor) -> torch.Tensor:
    """Ids by totals descending, ties by ascending id (planner.py:42-45). int64 CUDA."""
    lib = _lib.lib()
    n = totals.numel()
    if n and int(totals.min().item()) < 0:
        raise ValueError("hotness totals must be non-negative")
    order = torch.empty(n, dtype=torch.int64, device="cuda")
    if n:
        tb = lib.gc_descending_order_temp_bytes(n)
        tmp = _temp(tb)
        _lib.check(lib.gc_descending_order(totals.data_ptr(), n, order.data_ptr(), tmp.data_ptr(), tb,
                                           _lib.stream_handle()), "descending_order")
    return order


def hotness_descending_order(totals) -> np.ndarray:
    return device_descending_order(_dev_i64(totals)).cpu().numpy()


def device_colsum_argmax(rows: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Column sums and first argmax over the K rows of a [K, n] int64 CUDA tensor."""
    lib = _lib.lib()
    k, n = rows.shape
    totals = torch.empty(n, dtype=torch.int64, device="cuda")
    owner = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(lib.gc_colsum_argmax(rows.data_ptr(), k, n, totals.data_ptr(), owner.data_ptr(), _lib.stream_handle()),
               "colsum_argmax")
    return totals, owner


def device_distribute(order: torch.Tensor, length: int, owner: torch.Tensor, k: int) -> list[torch.Tensor]:
    """distribute_prefix on the device: stable split of order[:length] by owner."""
    lib = _lib.lib()
    out = torch.empty(max(length, 1), dtype=torch.int64, device="cuda")
    counts = torch.zeros(k, dtype=torch.int64, device="cuda")
    tb = lib.gc_distribute_prefix_temp_bytes(length, k)
    tmp = _temp(tb)
    _lib.check(lib.gc_distribute_prefix(order.data_ptr(), length, owner.data_ptr(), k, out.data_ptr(),
                                        counts.data_ptr(), tmp.data_ptr(), tb, _lib.stream_handle()), "distribute")
    c = counts.cpu().numpy()
    starts = np.concatenate([[0], np.cumsum(c)])
    return [out[starts[g] : starts[g + 1]] for g in range(k)]


@dataclass(frozen=True)
class CandidateOrders:
    """Ranked cache candidates of one clique (planner.py:21-39); arrays are numpy,
    device copies are kept for the plan search."""

    clique_id: int
    topo_totals: np.ndarray
    feat_totals: np.ndarray
    topo_order: np.ndarray
    feat_order: np.ndarray
    topo_owner: np.ndarray
    feat_owner: np.ndarray
    gpu_topo_queues: tuple[np.ndarray, ...]
    gpu_feat_queues: tuple[np.ndarray, ...]
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    def device(self, name: str) -> torch.Tensor:
        t = self._device.get(name)
        if t is None:
            arr = getattr(self, name)
            t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
            self._device[name] = t
        return t


def build_candidate_orders(hotness: HotnessMatrices) -> CandidateOrders:
    """Clique totals, CSLP rankings, first-argmax owners and per-GPU queues (planner.py:48-67)."""
    k = hotness.clique_size
    dev = {}
    out = {}
    for kind, rows in (("topo", hotness.topo_hotness), ("feat", hotness.feat_hotness)):
        r = _dev_i64(rows)
        totals, owner = device_colsum_argmax(r)
        order = device_descending_order(totals)
        queues = device_distribute(order, order.numel(), owner, k)
        dev.update({f"{kind}_totals": totals, f"{kind}_order": order, f"{kind}_owner": owner})
        out[kind] = (totals.cpu().numpy(), order.cpu().numpy(), owner.cpu().numpy(),
                     tuple(q.cpu().numpy() for q in queues))
    return CandidateOrders(
        clique_id=hotness.clique_id,
        topo_totals=out["topo"][0], feat_totals=out["feat"][0],
        topo_order=out["topo"][1], feat_order=out["feat"][1],
        topo_owner=out["topo"][2], feat_owner=out["feat"][2],
        gpu_topo_queues=out["topo"][3], gpu_feat_queues=out["feat"][3],
        _device=dev,
    )


@dataclass(frozen=True)
class CachePlan:
    """Budget split (B, alpha) (planner.py:70-84)."""

    budget_bytes: int
    alpha: float
    topo_budget: float
    feat_budget: float

    @classmethod
    def from_alpha(cls, budget_bytes: int, alpha: float) -> "CachePlan":
        if not 0.0 <= alpha <= 1.0:
            raise ValueError("alpha must be in [0, 1]")
        topo = budget_bytes * alpha
        return cls(budget_bytes, alpha, topo, budget_bytes - topo)


def _topo_prefix_dev(orders: CandidateOrders, graph: CsrGraph, spec: HardwareSpec) -> torch.Tensor:
    lib = _lib.lib()
    order = orders.device("topo_order")
    n = order.numel()
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    if n:
        tb = lib.gc_order_scan_temp_bytes(n)
        tmp = _temp(tb)
        _lib.check(lib.gc_topo_prefix_bytes(graph.device().c_struct.row_offsets, order.data_ptr(), n,
                                            spec.uint32_bytes, spec.uint64_bytes, out.data_ptr(), tmp.data_ptr(), tb,
                                            _lib.stream_handle()), "topo_prefix_bytes")
    return out


def _hot_prefix_dev(totals: torch.Tensor, order: torch.Tensor) -> torch.Tensor:
    lib = _lib.lib()
    n = order.numel()
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    if n:
        tb = lib.gc_order_scan_temp_bytes(n)
        tmp = _temp(tb)
        _lib.check(lib.gc_hot_prefix(totals.data_ptr(), order.data_ptr(), n, out.data_ptr(), tmp.data_ptr(), tb,
                                     _lib.stream_handle()), "hot_prefix")
    return out


def _searchsorted(prefix: torch.Tensor, budgets: np.ndarray) -> np.ndarray:
    lib = _lib.lib()
    b = torch.from_numpy(np.ascontiguousarray(budgets, dtype=np.float64)).cuda()
    out = torch.empty(len(budgets), dtype=torch.int64, device="cuda")
    _lib.check(lib.gc_searchsorted_right(prefix.data_ptr(), prefix.numel(), b.data_ptr(), len(budgets),
                                         out.data_ptr(), _lib.stream_handle()), "searchsorted")
    return out.cpu().numpy()


def topo_prefix_bytes(orders: CandidateOrders, graph: CsrGraph, spec: HardwareSpec) -> np.ndarray:
    """Cumulative neighbour-list + row-pointer bytes along the topology order (planner.py:87-90)."""
    return _topo_prefix_dev(orders, graph, spec).cpu().numpy()


def feat_prefix_bytes(orders: CandidateOrders, feat: FeatureSpec) -> np.ndarray:
    """(i+1) * row bytes (planner.py:93-95)."""
    return np.arange(1, len(orders.feat_order) + 1, dtype=np.int64) * feat.row_bytes


def _feat_prefix_dev(n: int, feat: FeatureSpec) -> torch.Tensor:
    return torch.arange(1, n + 1, dtype=torch.int64, device="cuda") * feat.row_bytes


def boundary_topology(orders: CandidateOrders, topo_budget: float, graph: CsrGraph, spec: HardwareSpec,
                      prefix: np.ndarray | None = None) -> int:
    """Longest topology prefix within the budget (planner.py:98-109)."""
    if topo_budget < 0:
        raise ValueError("budget must be >= 0")
    if prefix is not None:
        return int(np.searchsorted(prefix, topo_budget, side="right"))
    return int(_searchsorted(_topo_prefix_dev(orders, graph, spec), np.array([topo_budget]))[0])


def boundary_feature(orders: CandidateOrders, feat_budget: float, feat: FeatureSpec) -> int:
    """Feature rows within the budget, same float compare as the topology side (planner.py:112-121)."""
    if feat_budget < 0:
        raise ValueError("budget must be >= 0")
    return int(_searchsorted(_feat_prefix_dev(len(orders.feat_order), feat), np.array([feat_budget]))[0])


def feature_row_transactions(feat: FeatureSpec, spec: HardwareSpec) -> int:
    """ceil(row bytes / cache line) (planner.py:124-126)."""
    return -(-feat.row_bytes // spec.cache_line_bytes)


@dataclass(frozen=True)
class TrafficEstimate:
    """Predicted per-epoch PCIe transactions (planner.py:129-139)."""

    sampling_txns: float
    feature_txns: int
    total_txns: float
    topo_reduction: float
    feature_misses: int
    topo_prefix_len: int
    feat_prefix_len: int


def _estimate_at(b_t, b_f, t_pre, t_tot, f_pre, f_tot, txn_total, row_txns) -> TrafficEstimate:
    """Eqs. 4/5/7/8 with one correctly rounded division (planner.py:142-169)."""
    if t_tot > 0:
        reduction = t_pre / t_tot
        sampling = txn_total * (t_tot - t_pre) / t_tot
    else:
        reduction = 0.0
        sampling = float(txn_total)
    misses = f_tot - f_pre
    feature = row_txns * misses
    return TrafficEstimate(sampling, feature, sampling + feature, reduction, misses, b_t, b_f)


def estimate_traffic(orders: CandidateOrders, plan: CachePlan, graph: CsrGraph, feat: FeatureSpec,
                     spec: HardwareSpec, sampling_txn_total: int) -> TrafficEstimate:
    """Cost-model traffic of one (B, alpha) plan (planner.py:172-199)."""
    b_t = boundary_topology(orders, plan.topo_budget, graph, spec)
    b_f = boundary_feature(orders, plan.feat_budget, feat)
    t_cum = _hot_prefix_dev(orders.device("topo_totals"), orders.device("topo_order"))
    f_cum = _hot_prefix_dev(orders.device("feat_totals"), orders.device("feat_order"))
    t_pre = int(t_cum[b_t - 1].item()) if b_t else 0
    f_pre = int(f_cum[b_f - 1].item()) if b_f else 0
    t_tot = int(t_cum[-1].item()) if t_cum.numel() else 0
    f_tot = int(f_cum[-1].item()) if f_cum.numel() else 0
    return _estimate_at(b_t, b_f, t_pre, t_tot, f_pre, f_tot, int(sampling_txn_total),
                        feature_row_transactions(feat, spec))


def alpha_grid(delta_alpha: float) -> list[float]:
    """{0, d, 2d, ...} with 0 and 1 included (planner.py:202-212)."""
    if not 0.0 < delta_alpha <= 1.0:
        raise ValueError("delta_alpha must be in (0, 1]")
    steps = int(math.floor(1.0 / delta_alpha + 1e-9))
    grid = [i * delta_alpha for i in range(steps + 1)]
    if grid[-1] > 1.0:
        grid[-1] = 1.0
    if grid[-1] < 1.0 - 1e-12:
        grid.append(1.0)
    return grid


def search_optimal_plan(orders: CandidateOrders, budget_bytes: int, delta_alpha: float, graph: CsrGraph,
                        feat: FeatureSpec, spec: HardwareSpec, sampling_txn_total: int, *,
                        bandwidths=None) -> tuple[CachePlan, TrafficEstimate]:
    """Alpha sweep from one pair of device scans and batched boundary searches; the
    winner is the first strict minimum, i.e. the smallest alpha (planner.py:215-261).

    bandwidths (a bandwidth.MeasuredBandwidths): minimise the host-tier time predicted
    from bandwidths measured on the box (bandwidth.estimate_seconds) instead of the
    reference's transaction count; the returned estimate is the winner's
    TrafficEstimate either way."""
    return _search(orders, budget_bytes, delta_alpha, graph, feat, spec, sampling_txn_total, bandwidths)[:2]


def sweep_alpha(orders: CandidateOrders, budget_bytes: int, delta_alpha: float, graph: CsrGraph,
                feat: FeatureSpec, spec: HardwareSpec, sampling_txn_total: int, bandwidths=None
                ) -> list[tuple[float, TrafficEstimate, float | None]]:
    """(alpha, TrafficEstimate, predicted seconds or None) for every grid point — the
    predicted side of the reference's alpha sweep (cli.py:276-340)."""
    return _search(orders, budget_bytes, delta_alpha, graph, feat, spec, sampling_txn_total, bandwidths)[2]


def _search(orders, budget_bytes, delta_alpha, graph, feat, spec, sampling_txn_total, bandwidths):
    grid = np.array(alpha_grid(delta_alpha))
    topo_budgets = grid * budget_bytes
    feat_budgets = budget_bytes - topo_budgets
    s_topo = _topo_prefix_dev(orders, graph, spec)
    s_feat = _feat_prefix_dev(len(orders.feat_order), feat)
    b_t = _searchsorted(s_topo, topo_budgets)
    b_f = _searchsorted(s_feat, feat_budgets)
    t_cum = _hot_prefix_dev(orders.device("topo_totals"), orders.device("topo_order"))
    f_cum = _hot_prefix_dev(orders.device("feat_totals"), orders.device("feat_order"))
    # hot_cum[b] = inclusive scan at b-1 (0 for an empty prefix): gather the 2 x |grid| values
    idx_t = torch.from_numpy(np.maximum(b_t - 1, 0)).cuda()
    idx_f = torch.from_numpy(np.maximum(b_f - 1, 0)).cuda()
    t_at = np.where(b_t > 0, t_cum[idx_t].cpu().numpy() if t_cum.numel() else 0, 0)
    f_at = np.where(b_f > 0, f_cum[idx_f].cpu().numpy() if f_cum.numel() else 0, 0)
    t_tot = int(t_cum[-1].item()) if t_cum.numel() else 0
    f_tot = int(f_cum[-1].item()) if f_cum.numel() else 0
    row_txns = feature_row_transactions(feat, spec)
    best, best_idx, best_cost = None, -1, None
    points = []
    for i in range(len(grid)):
        est = _estimate_at(int(b_t[i]), int(b_f[i]), int(t_at[i]), t_tot, int(f_at[i]), f_tot,
                           int(sampling_txn_total), row_txns)
        secs = None
        if bandwidths is not None:
            from .bandwidth import estimate_seconds

            secs = estimate_seconds(est, feat, spec, bandwidths)
        points.append((float(grid[i]), est, secs))
        cost = est.total_txns if bandwidths is None else secs
        if best is None or cost < best_cost:
            best, best_idx, best_cost = est, i, cost
    return CachePlan.from_alpha(budget_bytes, float(grid[best_idx])), best, points


def distribute_prefix(prefix: np.ndarray, owner_local: np.ndarray, clique_size: int) -> list[np.ndarray]:
    """Split a ranked prefix into per-GPU queues by owner, keeping order (planner.py:264-267)."""
    pre = _dev_i64(prefix)
    own = torch.from_numpy(np.ascontiguousarray(owner_local, dtype=np.int32)).cuda()
    return [q.cpu().numpy() for q in device_distribute(pre, pre.numel(), own, clique_size)]


@dataclass
class CacheAssignment:
    """Per-GPU cache contents, global GPU ids (planner.py:270-286)."""

    num_gpus: int
    topo_vertices: list[np.ndarray]
    feat_vertices: list[np.ndarray]
    topo_bytes: list[int]
    feat_bytes: list[int]

    @classmethod
    def empty(cls, num_gpus: int) -> "CacheAssignment":
        nothing = [np.empty(0, dtype=np.int64) for _ in range(num_gpus)]
        return cls(num_gpus, nothing, list(nothing), [0] * num_gpus, [0] * num_gpus)

    def gpu_bytes(self, gpu: int) -> int:
        return self.topo_bytes[gpu] + self.feat_bytes[gpu]


def materialize_assignment(orders_by_clique: list[CandidateOrders], plans: list[CachePlan], layout: CliqueLayout,
                           graph: CsrGraph, feat: FeatureSpec, spec: HardwareSpec) -> CacheAssignment:
    """Cached prefixes placed on their owner GPUs, byte accounting, budget check
    (planner.py:289-319)."""
    if len(orders_by_clique) != layout.clique_count or len(plans) != layout.clique_count:
        raise ValueError("need one CandidateOrders and one CachePlan per clique")
    out = CacheAssignment.empty(layout.num_gpus)
    deg = graph.out_degrees
    for ci, members in enumerate(layout.cliques):
        orders, plan = orders_by_clique[ci], plans[ci]
        b_t = boundary_topology(orders, plan.topo_budget, graph, spec)
        b_f = boundary_feature(orders, plan.feat_budget, feat)
        tq = device_distribute(orders.device("topo_order"), b_t, orders.device("topo_owner"), len(members))
        fq = device_distribute(orders.device("feat_order"), b_f, orders.device("feat_owner"), len(members))
        total = 0
        for li, gpu in enumerate(members):
            tv, fv = tq[li].cpu().numpy(), fq[li].cpu().numpy()
            t_bytes = int((deg[tv] * spec.uint32_bytes + spec.uint64_bytes).sum())
            f_bytes = len(fv) * feat.row_bytes
            out.topo_vertices[gpu], out.feat_vertices[gpu] = tv, fv
            out.topo_bytes[gpu], out.feat_bytes[gpu] = t_bytes, f_bytes
            total += t_bytes + f_bytes
        if total > plan.budget_bytes:
            raise AssertionError("materialized clique cache exceeds its budget")
    return out


def plan_report(layout: CliqueLayout, plans: list[CachePlan], estimates: list[TrafficEstimate], delta_alpha: float,
                tablet_sizes: list[list[int]] | None = None) -> dict:
    """JSON-ready per-clique plan summary (planner.py:322-351)."""
    cliques = []
    for ci in range(layout.clique_count):
        plan, est = plans[ci], estimates[ci]
        entry = {"clique": ci, "alpha": plan.alpha, "topo_budget_bytes": plan.topo_budget,
                 "feat_budget_bytes": plan.feat_budget, "topo_prefix_len": est.topo_prefix_len,
                 "feat_prefix_len": est.feat_prefix_len, "sampling_txns": est.sampling_txns,
                 "feature_txns": est.feature_txns, "total_txns": est.total_txns}
        if tablet_sizes is not None:
            entry["tablet_sizes"] = tablet_sizes[ci]
        cliques.append(entry)
    return {"delta_alpha": delta_alpha, "alpha_grid_points": len(alpha_grid(delta_alpha)), "cliques": cliques}
