"""Legion's partitioned clique cache, one process per GPU (the north-star configuration).

The whole 8xB200 box is one NVSwitch clique, so the cache is partitioned over its
GPUs rather than replicated: CSLP gives every cached vertex exactly one owner GPU —
the first argmax of the clique's per-GPU hotness rows (planner.py:48-67, :289-319) —
and a GPU reads a vertex it does not own from that owner's HBM over NVLink, else from
the host (the tier rule, simulator.py:161-202). Per rank, in order:

  1. presampling of this rank's own tablet (K1/K2/K3/K5; sampling.py:247-289 restricted
     to row `local_idx`) -> H_T row, H_F row, N_TSUM share, all in HBM
  2. the clique's one exchange step: all-reduce SUM of the rows, all-reduce MAX of
     (row << 3 | 7 - rank) for the lowest-index argmax, all-reduce SUM of N_TSUM
     (distributed.merge_hotness) -> identical CandidateOrders on every rank
  3. alpha search + materialize_assignment (K6/K7; deterministic, so every rank derives
     the same plan and assignment without a broadcast)
  4. this rank fills only its own slabs: neighbour lists by K8 from the full CSR,
     feature rows by K4 from the node-shared pinned host table (hostmem)
  5. CUDA IPC handles of the slabs are all-gathered and the peers' mapped
     (distributed.exchange_addresses), so the sampler and the gather read peer HBM
     with one-sided loads; there is no collective in the per-batch loop.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import planner as PL
from .cache import FeatureStore, TopologyStore
from .distributed import candidate_orders_from_rows, exchange_addresses, sum_over_ranks
from .graph import CsrGraph, FeatureSpec
from .hardware import CliqueLayout, HardwareSpec
from .rng import KeyedRng
from .sampling import DeviceHotness, EpochRunner, SamplingConfig


@dataclass
class CliqueRank:
    """One rank's view of the partitioned clique cache."""

    rank: int
    world: int
    orders: PL.CandidateOrders
    plan: PL.CachePlan
    estimate: PL.TrafficEstimate
    assignment: PL.CacheAssignment
    sampling_txn_total: int
    topology: TopologyStore
    features: FeatureStore
    presample_batches: int  # batches of the whole clique behind the plan (for N_total per batch)

    def predicted_pcie_txn_per_batch(self) -> float:
        """The reference plan's PCIe prediction per batch: N_total / clique batches
        (planner.py:142-169; N_TSUM and the hotness counted presample_batches batches)."""
        return self.estimate.total_txns / max(self.presample_batches, 1)


def presample_rows(graph: CsrGraph, pool: np.ndarray, clique_idx: int, local_idx: int, cfg: SamplingConfig,
                   spec: HardwareSpec) -> tuple[DeviceHotness, int]:
    """This GPU's row of run_presampling (sampling.py:247-289): cfg.presample_epochs
    epochs of its own tablet with the streams root.derive(epoch, clique, gpu) ->
    (device counters, batches sampled)."""
    hot = DeviceHotness(graph.num_vertices, spec)
    pool = np.asarray(pool, dtype=np.int64)
    if len(pool) == 0:
        warnings.warn(f"empty training tablet for gpu {local_idx}; its hotness rows stay zero")
        return hot, 0
    runner = EpochRunner(graph, cfg, len(pool))
    root = KeyedRng(cfg.seed)
    batches = 0
    for epoch in range(cfg.presample_epochs):
        batches += runner.run(pool, root.derive(epoch, clique_idx, local_idx), hot)
    return hot, batches


def build_clique_cache(graph: CsrGraph, pool: np.ndarray, layout: CliqueLayout, cfg: SamplingConfig,
                       feat: FeatureSpec, spec: HardwareSpec, host_table: torch.Tensor, *, rank: int, world: int,
                       group=None, delta_alpha: float = 0.01, host_full_topology: bool = True,
                       bandwidths=None) -> CliqueRank:
    """Collective over the clique's processes (rank r drives GPU r of the single clique;
    `pool` is its own tablet, `host_table` the node-shared pinned fp32 [n, D] table).
    Every rank returns its CliqueRank; the stores read peer slabs through CUDA IPC."""
    if layout.clique_count != 1 or layout.num_gpus != world:
        raise ValueError("one process per GPU of a single clique: layout must be block_layout(world, world)")
    clique_idx, local_idx = layout.gpu_position(rank)
    distributed = dist.is_initialized()
    if world > 1 and not distributed:
        raise ValueError("world > 1 needs an initialised torch.distributed process group")
    backend = dist.get_backend(group) if distributed else "none"
    # 1. presampling of this rank's tablet
    hot, my_batches = presample_rows(graph, pool, clique_idx, local_idx, cfg, spec)
    # 2. hotness merge (the one exchange step): rows on the collective backend's device
    on = (lambda t: t) if backend == "nccl" else (lambda t: t.cpu())
    orders = candidate_orders_from_rows(on(hot.edge_traversals), on(hot.feat_lookups), local_idx, world,
                                        clique_idx, group)
    txn_total = sum_over_ranks(int(hot.txn_total.item()), group)
    batches = sum_over_ranks(my_batches, group)
    del hot
    # 3. plan + assignment: identical on every rank
    plan, est = PL.search_optimal_plan(orders, spec.clique_budget_bytes, delta_alpha, graph, feat, spec, txn_total,
                                       bandwidths=bandwidths)
    asg = PL.materialize_assignment([orders], [plan], layout, graph, feat, spec)
    # 4. this rank's slabs only
    t_offs, t_cols = TopologyStore.build_slab(graph, asg.topo_vertices[rank], host_full_topology)
    f_slab = FeatureStore.build_slab(host_table, asg.feat_vertices[rank])
    torch.cuda.synchronize()
    # 5. peers' slabs mapped over NVLink (CUDA IPC)
    addrs = exchange_addresses([t_offs, t_cols, f_slab], rank, world, group)
    topo_slabs = [(t_offs, t_cols) if g == rank else (a[0], a[1]) for g, a in enumerate(addrs)]
    feat_slabs = [f_slab if g == rank else a[2] for g, a in enumerate(addrs)]
    topology = TopologyStore(graph, asg.topo_vertices, rank, host_full=host_full_topology, peer_slabs=topo_slabs)
    features = FeatureStore.from_assignment(host_table, asg.feat_vertices, rank, peer_slabs=feat_slabs)
    # keep the own slabs alive with the stores; every rank must have mapped before use
    features._keep.append((t_offs, t_cols))
    if distributed:
        dist.barrier(group)
    return CliqueRank(rank, world, orders, plan, est, asg, txn_total, topology, features, batches)
