"""Training-vertex sharding across the GPUs of a clique (partition.py of the reference).

Host-side preprocessing that stays on the host (north star). On one 8xB200 NVSwitch
clique the inter-clique LDG level collapses (num_parts == 1 returns all zeros,
partition.py:100-101), so only the intra-clique tablet split and its binding to
GPUs are needed to produce the per-GPU seed pools of the data path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import CsrGraph, TrainingSet
from .hardware import CliqueLayout


def _mix64_np(x: np.ndarray) -> np.ndarray:
    # splitmix64 finalizer (rng.py:34-42) for the host-side tablet hash
    x = x.astype(np.uint64, copy=True)
    x ^= x >> np.uint64(30)
    x *= np.uint64(0xBF58476D1CE4E5B9)
    x ^= x >> np.uint64(27)
    x *= np.uint64(0x94D049BB133111EB)
    x ^= x >> np.uint64(31)
    return x


@dataclass(frozen=True)
class Partitioning:
    """Vertex -> partition (partition.py:21-33)."""

    assignments: np.ndarray
    num_parts: int

    def __post_init__(self):
        a = np.asarray(self.assignments, dtype=np.int32)
        a.setflags(write=False)
        object.__setattr__(self, "assignments", a)

    def part_sizes(self) -> np.ndarray:
        return np.bincount(self.assignments, minlength=self.num_parts)


def single_clique_partitioning(graph: CsrGraph) -> Partitioning:
    """partition_inter_clique with num_parts == 1 (partition.py:100-101)."""
    return Partitioning(np.zeros(graph.num_vertices, dtype=np.int32), 1)


@dataclass(frozen=True)
class TabletAssignment:
    """Per-clique, per-GPU disjoint training pools (partition.py:166-170)."""

    tablets: tuple[tuple[np.ndarray, ...], ...]


def split_intra_clique(training: TrainingSet, partitioning: Partitioning, layout: CliqueLayout) -> TabletAssignment:
    """Hash split mix64(v) % K_g, then round-robin rebalance to sizes differing by <= 1
    (partition.py:176-205). Vectorised: kept ids are each slot's first `quota`
    members in training order; the surplus, concatenated slot by slot, refills the
    short slots from its front — the same lists the reference's pop(0) loop builds."""
    if partitioning.num_parts != layout.clique_count:
        raise ValueError("partition count must equal the clique count")
    k = layout.clique_size
    out = []
    for clique in range(layout.clique_count):
        ids = training.vertex_ids[partitioning.assignments[training.vertex_ids] == clique]
        slot = (_mix64_np(ids.astype(np.uint64)) % np.uint64(k)).astype(np.int64)
        base, rem = divmod(len(ids), k)
        quota = np.array([base + (1 if t < rem else 0) for t in range(k)], dtype=np.int64)
        members = [ids[slot == t] for t in range(k)]
        keep = [m[: quota[t]] for t, m in enumerate(members)]
        surplus = np.concatenate([m[quota[t] :] for t, m in enumerate(members)] + [np.empty(0, np.int64)])
        pos = 0
        lists = []
        for t in range(k):
            need = int(quota[t] - len(keep[t]))
            lists.append(np.concatenate([keep[t], surplus[pos : pos + need]]).astype(np.int64))
            pos += need
        out.append(tuple(lists))
    return TabletAssignment(tuple(out))


def assign_tablets(tablets: TabletAssignment, layout: CliqueLayout) -> list[np.ndarray]:
    """Tablet [i][j] -> j-th GPU of clique i (partition.py:208-218)."""
    if len(tablets.tablets) != layout.clique_count:
        raise ValueError("tablet cliques do not match layout")
    pools = [np.empty(0, dtype=np.int64)] * layout.num_gpus
    for ci, members in enumerate(layout.cliques):
        if len(tablets.tablets[ci]) != len(members):
            raise ValueError("tablet count does not match GPUs in clique")
        for li, gpu in enumerate(members):
            pools[gpu] = tablets.tablets[ci][li]
    return pools
