"""Unified feature cache and the three-tier gather (K4).

The reference stores no feature values; it only defines which tier
serves a row — local cache, the lowest-index clique peer holding it, else the CPU
(account_assignment, simulator.py:161-202) — and materialize_assignment
(planner.py:289-319) decides cache contents. This module builds the physical
layout for one GPU from a CacheAssignment:

  location table  u32 [n]: (owner_gpu << 28) | slot, or GC_TIER_HOST
  slabs           fp32 [rows_g, D] per clique GPU: the local one in this GPU's HBM,
                  the others mapped from the peers (CUDA IPC handles across processes,
                  or device pointers when one process drives several GPUs)
  host tier       the full fp32 table in pinned, mapped host memory (UVA over PCIe)

and gathers rows with gc_gather: 16-byte vector loads, one thread per vector.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph, FeatureSpec

TIER_NAMES = ("local", "peer", "host")


class TopologyStore:
    """Tiered neighbour lists of one GPU (Legion's topology cache).

    CacheAssignment.topo_vertices of the clique decide the slabs: GPU g's compact CSR
    holds the lists CSLP placed on g (in priority order); everything else is read
    from the full CSR in pinned, mapped host memory over PCIe (or from an HBM copy
    when host_full=False). Slabs are filled by the K8 copy kernel from the full CSR.
    With peer_slabs=None every slab of the clique is built in this process on the
    current device; otherwise peer_slabs[g] = (offsets address, cols address) mapped
    from GPU g."""

    def __init__(self, graph: CsrGraph, topo_vertices: list[np.ndarray], self_rank: int, host_full: bool = True,
                 peer_slabs: list | None = None):
        lib = _lib.lib()
        n = graph.num_vertices
        k = len(topo_vertices)
        if not 0 <= self_rank < k or k > _lib.GC_MAX_PEERS:
            raise ValueError("self_rank must index the clique (at most 8 GPUs)")
        self.full = graph.device("host" if host_full else "hbm")
        loc = np.full(n, _lib.GC_TIER_HOST, dtype=np.uint32)
        self.slabs: list = []
        for g, verts in enumerate(topo_vertices):
            verts = np.asarray(verts, dtype=np.int64)
            if len(verts) >= 1 << 28:
                raise ValueError("at most 2^28 cached neighbour lists per GPU")
            if len(verts) and (loc[verts] != _lib.GC_TIER_HOST).any():
                raise ValueError("a vertex's topology is cached on two GPUs; the clique cache is partitioned")
            loc[verts] = (np.uint32(g) << np.uint32(28)) | np.arange(len(verts), dtype=np.uint32)
            if peer_slabs is not None and (g != self_rank or peer_slabs[g] is not None):
                self.slabs.append(peer_slabs[g])  # mapped peer slab, or this GPU's prebuilt one
                continue
            self.slabs.append(self.build_slab(graph, verts, host_full))
        self.location = torch.from_numpy(loc.view(np.int32)).cuda()
        self.tier_reads = torch.zeros(7, dtype=torch.int64, device="cuda")
        t = _lib.GcTopology()
        t.full = self.full.c_struct
        t.location = self.location.data_ptr()
        for g, slab in enumerate(self.slabs):
            o, c = slab
            t.slab_offsets[g] = o if isinstance(o, int) else o.data_ptr()
            t.slab_cols[g] = c if isinstance(c, int) else c.data_ptr()
        t.self_rank = self_rank
        t.full_on_host = 1 if host_full else 0
        t.tier_reads = self.tier_reads.data_ptr()
        self.c_struct = t
        self.self_rank = self_rank

    @staticmethod
    def build_slab(graph: CsrGraph, verts: np.ndarray, host_full: bool = True) -> tuple:
        """This GPU's compact CSR of the lists in `verts` (priority order), filled on the
        device by K8 from the full CSR (pinned host or HBM): (offsets u64 as int64
        [len+1], cols int32 [max(1, edges)])."""
        verts = np.asarray(verts, dtype=np.int64)
        full = graph.device("host" if host_full else "hbm")
        offs = np.zeros(len(verts) + 1, dtype=np.uint64)
        np.cumsum(graph.out_degrees[verts], out=offs[1:])
        d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
        d_cols = torch.empty(max(int(offs[-1]), 1), dtype=torch.int32, device="cuda")
        d_ids = torch.from_numpy(verts).cuda()
        _lib.check(_lib.lib().gc_csr_extract(full.c_struct, d_ids.data_ptr(), len(verts), d_offs.data_ptr(),
                                             d_cols.data_ptr(), _lib.stream_handle()), "csr_extract")
        return d_offs, d_cols

    def tier_counts(self) -> dict:
        v = self.tier_reads.cpu().numpy()
        out = {f"{what}_{tier}": int(v[i * 3 + j]) for i, what in enumerate(("reads", "edges"))
               for j, tier in enumerate(TIER_NAMES)}
        out["host_txn"] = int(v[6])  # PCIe transactions, the unit of TrafficReport.sampling_cpu_txn
        return out

    def reset_counters(self) -> None:
        self.tier_reads.zero_()

    def host_bytes(self) -> int:
        """PCIe payload of host-tier list reads so far: a 16-byte row-offset pair per read
        plus 4 bytes per sampled column."""
        v = self.tier_reads.cpu().numpy()
        return int(16 * v[2] + 4 * v[5])


@dataclass
class FeatureStore:
    """Feature rows of one GPU's view of the clique cache."""

    spec: FeatureSpec
    self_rank: int
    num_ranks: int
    location: torch.Tensor | None  # int32 view of u32 [n]; None = fully resident local table
    slabs: list  # per clique rank: torch.Tensor (local/same-process) or int address (IPC-mapped)
    host_table: torch.Tensor | None = None  # pinned fp32 [n, D]
    tier_rows: torch.Tensor = field(default=None)  # u64[3] cumulative rows served per tier
    _keep: list = field(default_factory=list, repr=False)
    _defer: dict = field(default_factory=dict, repr=False)  # stream handle -> deferred-row list buffer

    def __post_init__(self):
        if self.tier_rows is None:
            self.tier_rows = torch.zeros(3, dtype=torch.int64, device="cuda")
        s = _lib.GcFeatureStore()
        s.row_bytes = self.spec.row_bytes
        s.self_rank = self.self_rank
        s.num_ranks = self.num_ranks
        s.location = _lib.ptr(self.location)
        for g, slab in enumerate(self.slabs):
            s.slabs[g] = slab if isinstance(slab, int) else (slab.data_ptr() if slab is not None else None)
        s.host_rows = _lib.ptr(self.host_table)
        self.c_struct = s

    # ---------------------------------------------------------------- builders
    @classmethod
    def resident(cls, table: torch.Tensor) -> "FeatureStore":
        """Whole table in local HBM (BASELINE config 2: fully HBM-cached)."""
        if table.dtype != torch.float32 or not table.is_cuda or table.dim() != 2:
            raise ValueError("table must be a 2-D float32 CUDA tensor")
        return cls(FeatureSpec(table.shape[1]), 0, 1, None, [table.contiguous()])

    @classmethod
    def from_assignment(cls, host_table: np.ndarray | torch.Tensor, feat_vertices: list[np.ndarray], self_rank: int,
                        peer_slabs: list | None = None) -> "FeatureStore":
        """Cache laid out from CacheAssignment.feat_vertices of one clique (local ids).

        Slot order is the assignment's priority order. When peer_slabs is None every
        slab of the clique is built in this process on the current device (single
        process driving the whole clique, or a test of the peer path on one GPU);
        otherwise peer_slabs[g] is the mapped address of GPU g's slab."""
        host = torch.as_tensor(host_table)
        if host.dtype != torch.float32 or host.dim() != 2:
            raise ValueError("host_table must be float32 [n, D]")
        n, dim = host.shape
        k = len(feat_vertices)
        if not 0 <= self_rank < k or k > _lib.GC_MAX_PEERS:
            raise ValueError("self_rank must index the clique (at most 8 GPUs)")
        loc = np.full(n, _lib.GC_TIER_HOST, dtype=np.uint32)
        for g, verts in enumerate(feat_vertices):
            verts = np.asarray(verts, dtype=np.int64)
            if len(verts) >= 1 << 28:
                raise ValueError("at most 2^28 cached rows per GPU")
            if len(verts) and (loc[verts] != _lib.GC_TIER_HOST).any():
                raise ValueError("a vertex is cached on two GPUs; the clique cache is partitioned")
            loc[verts] = (np.uint32(g) << np.uint32(28)) | np.arange(len(verts), dtype=np.uint32)
        pinned = host.contiguous().pin_memory() if not host.is_pinned() else host
        slabs: list = []
        for g, verts in enumerate(feat_vertices):
            if peer_slabs is not None and (g != self_rank or peer_slabs[g] is not None):
                slab = peer_slabs[g]  # mapped peer slab (address), or this GPU's prebuilt one
                slabs.append(slab if isinstance(slab, torch.Tensor) else int(slab))
                continue
            slabs.append(cls.build_slab(pinned, verts))
        location = torch.from_numpy(loc.view(np.int32)).cuda()
        return cls(FeatureSpec(dim), self_rank, k, location, slabs, pinned)

    @staticmethod
    def build_slab(host_table: torch.Tensor, verts: np.ndarray, chunk: int = 1 << 20) -> torch.Tensor:
        """This GPU's feature slab: rows X[verts] (priority order) pulled from the pinned,
        mapped host table by the K4 gather itself (the table read as a resident tier
        through UVA), so a multi-GB fill moves at PCIe speed with no host-side copy."""
        verts = np.asarray(verts, dtype=np.int64)
        dim = host_table.shape[1]
        slab = torch.empty((max(len(verts), 1), dim), dtype=torch.float32, device="cuda")
        if not len(verts):
            return slab
        if not host_table.is_pinned():
            raise ValueError("host_table must be pinned (mapped) memory")
        src = FeatureStore(FeatureSpec(dim), 0, 1, None, [int(host_table.data_ptr())])
        ids = torch.from_numpy(verts.astype(np.uint32).view(np.int32)).cuda()
        for c0 in range(0, len(verts), chunk):
            c1 = min(len(verts), c0 + chunk)
            cnt = torch.tensor([c1 - c0], dtype=torch.int32, device="cuda")
            src.gather(ids[c0:c1].view(1, -1), cnt, slab[c0:c1].view(1, c1 - c0, dim))
        return slab

    # ---------------------------------------------------------------- gather
    def gather(self, ids: torch.Tensor, counts: torch.Tensor, out: torch.Tensor, num_batches: int | None = None,
               stream=None, deferred: bool = False, host_stream=None) -> torch.Tensor:
        """out[b, k] = X[ids[b, k]] for k < min(counts[b], out.shape[1]) (K4).

        ids: int32 [W, cap] CUDA, counts: int32 [W] CUDA, out: float32 [W, rows, D].
        deferred: host-tier rows are copied by a second small-grid kernel
        (gc_gather_deferred) — on `host_stream` when given — so the PCIe-bound part
        overlaps other streams' work; `stream` is ordered after it either way."""
        lib = _lib.lib()
        if ids.dim() == 1:
            ids, out = ids.view(1, -1), out.view(1, *out.shape)
        W = ids.shape[0] if num_batches is None else num_batches
        if out.shape[-1] * 4 != self.spec.row_bytes:
            raise ValueError("output row width does not match the feature store")
        s = _lib.stream_handle(stream)
        if deferred and self.host_table is not None and self.location is not None:
            need = int(lib.gc_gather_defer_bytes(out.shape[1], W))
            buf = self._defer.get(s)
            if buf is None or buf.numel() < need:
                buf = torch.empty(need, dtype=torch.uint8, device="cuda")
                self._defer[s] = buf  # one list per stream: concurrent lanes never share it
            _lib.check(
                lib.gc_gather_deferred(self.c_struct, ids.data_ptr(), ids.shape[1], counts.data_ptr(), out.shape[1],
                                       W, out.data_ptr(), out.shape[1], self.tier_rows.data_ptr(), buf.data_ptr(),
                                       buf.numel(), s, _lib.stream_handle(host_stream) if host_stream else None),
                "gather_deferred",
            )
            return out
        _lib.check(
            lib.gc_gather(self.c_struct, ids.data_ptr(), ids.shape[1], counts.data_ptr(), out.shape[1], W,
                          out.data_ptr(), out.shape[1], self.tier_rows.data_ptr(), s),
            "gather",
        )
        return out

    def tier_counts(self) -> dict:
        v = self.tier_rows.cpu().numpy()
        return {name: int(x) for name, x in zip(TIER_NAMES, v)}

    def reset_counters(self) -> None:
        self.tier_rows.zero_()


def gather_rows(store: FeatureStore, ids: np.ndarray) -> np.ndarray:
    """Host convenience: X[ids] through the device gather (ids int64 numpy)."""
    ids = np.asarray(ids, dtype=np.int64)
    d = torch.from_numpy(ids.astype(np.uint32).view(np.int32)).cuda().view(1, -1)
    cnt = torch.tensor([len(ids)], dtype=torch.int32, device="cuda")
    out = torch.empty((1, max(len(ids), 1), store.spec.dimension), dtype=torch.float32, device="cuda")
    store.gather(d, cnt, out)
    return out[0, : len(ids)].cpu().numpy()
