"""Hierarchical partitioning (partition.py of the reference): the inter-clique LDG
edge-cut split and the intra-clique training-vertex tablets.

Host-side preprocessing (north star). On one 8xB200 NVSwitch clique the
inter-clique level collapses (num_parts == 1 returns all zeros, partition.py:100-101);
for several cliques, and for the pagraph-plus comparison policy, the LDG placement
runs natively in the library (gc_partition_ldg: sequential greedy + refinement in
C++, BFS roots from the device permutation).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import CsrGraph, TrainingSet
from .hardware import CliqueLayout
from .rng import KeyedRng

ROLE_BFS_ROOTS = 0x5EED  # partition.py:53


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


def ldg_capacity(n: int, num_parts: int, epsilon: float) -> int:
    """Per-part vertex cap, int((1 + eps) * ceil(n / k)) and at least ceil(n / k)
    (partition.py:103-104)."""
    even = math.ceil(n / num_parts)
    return max(int((1.0 + epsilon) * even), even)


def ldg_assign(graph: CsrGraph, num_parts: int, capacity: int, root_order: np.ndarray, refine_passes: int = 2,
               lib: ctypes.CDLL | None = None) -> tuple[np.ndarray, np.ndarray]:
    """gc_partition_ldg over host arrays: (assignments int32 [n], per-pass cuts
    uint64 [passes, 2] before/after, zero rows for passes not run)."""
    n = graph.num_vertices
    roots = np.ascontiguousarray(root_order, dtype=np.int64)
    if roots.shape != (n,):
        raise ValueError("root_order must hold every vertex once")
    out = np.empty(n, dtype=np.int32)
    cuts = np.zeros((max(refine_passes, 1), 2), dtype=np.uint64)
    L = lib if lib is not None else _lib.lib()
    _lib.check(L.gc_partition_ldg(graph.row_offsets.ctypes.data, graph.col_indices.ctypes.data, n, graph.num_edges,
                                  roots.ctypes.data, num_parts, capacity, refine_passes, out.ctypes.data,
                                  cuts.ctypes.data), "partition_inter_clique")
    return out, cuts[: max(refine_passes, 0)]


def partition_inter_clique(graph: CsrGraph, num_parts: int, epsilon: float = 0.05, seed: int = 0,
                           refine_passes: int = 2) -> Partitioning:
    """Balanced edge-cut-minimising streaming partition, deterministic per seed
    (partition.py:85-130): BFS stream order from KeyedRng(seed).derive(0x5EED)'s
    permutation (device), then the native LDG placement + refinement."""
    n = graph.num_vertices
    if num_parts < 1:
        raise ValueError("num_parts must be >= 1")
    if num_parts > n:
        raise ValueError(f"num_parts {num_parts} exceeds num_vertices {n}")
    if epsilon < 0:
        raise ValueError("epsilon must be >= 0")
    if num_parts == 1:
        return Partitioning(np.zeros(n, dtype=np.int32), 1)
    roots = KeyedRng(seed).derive(ROLE_BFS_ROOTS).permutation(n)
    assignments, _ = ldg_assign(graph, num_parts, ldg_capacity(n, num_parts, epsilon), roots, refine_passes)
    return Partitioning(assignments, num_parts)


def edge_cut_ratio(graph: CsrGraph, partitioning: Partitioning) -> float:
    """Fraction of directed edges whose endpoints lie in different parts (partition.py:162-166)."""
    if graph.num_edges == 0:
        return 0.0
    a = partitioning.assignments
    src = np.repeat(np.arange(graph.num_vertices, dtype=np.int64), graph.out_degrees)
    return int(np.count_nonzero(a[src] != a[graph.col_indices.astype(np.int64)])) / graph.num_edges


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


def dump_partitioning(partitioning: Partitioning, path) -> None:
    """One "vertex part" line per vertex (partition.py:221-224)."""
    a = np.asarray(partitioning.assignments, dtype=np.int64)
    with open(path, "w", encoding="utf-8") as fh:
        np.savetxt(fh, np.stack([np.arange(len(a), dtype=np.int64), a], axis=1), fmt="%d")


def dump_tablets(tablets: TabletAssignment, layout: CliqueLayout, path) -> None:
    """One "vertex clique gpu_in_clique" line per training vertex, clique-major
    (partition.py:227-232)."""
    with open(path, "w", encoding="utf-8") as fh:
        for ci in range(layout.clique_count):
            for li in range(layout.clique_size):
                v = np.asarray(tablets.tablets[ci][li], dtype=np.int64)
                if len(v):
                    rows = np.stack([v, np.full(len(v), ci, np.int64), np.full(len(v), li, np.int64)], axis=1)
                    np.savetxt(fh, rows, fmt="%d")
