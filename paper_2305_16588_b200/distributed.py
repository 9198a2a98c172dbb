"""One process per GPU: the path's only exchange steps.

The per-batch loop needs no collective: every rank samples its own tablet with the
reference's per-(epoch, clique, gpu) streams (sampling.py:224-234) and reads peer
cache slabs one-sided over NVLink. Two things cross ranks:

1. the presampling hotness merge — the planner needs clique-wide column sums and the
   first-argmax owner over the clique's rows (planner.py:50-55). Each rank holds one
   row; sums are an all-reduce(SUM), and the lowest-index argmax is an
   all-reduce(MAX) over (hotness << 3) | (7 - local_rank): the max value wins and,
   among equal values, the smallest rank index (np.argmax picks the first maximum);
2. the cache slab addresses — each rank exports CUDA IPC handles of its slabs once and
   maps its peers' (gc_ipc_export / gc_ipc_import), so gathers read peer HBM directly.

Collectives go through torch.distributed (NCCL on GPUs, gloo for the CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

OWNER_BITS = 3  # up to 8 GPUs per clique
MAX_HOTNESS = (1 << (63 - OWNER_BITS)) - 1


def merge_hotness(topo_row: torch.Tensor, feat_row: torch.Tensor, local_rank: int, group=None):
    """All-reduce one rank's hotness rows into (topo_totals, topo_owner, feat_totals,
    feat_owner) on every rank. Rows are int64 on the backend's device."""
    out = []
    if not dist.is_initialized():  # a single-GPU clique: the row is the column sum, owner 0
        for row in (topo_row, feat_row):
            out += [row.clone(), torch.zeros(row.shape, dtype=torch.int32, device=row.device)]
        return tuple(out)
    for row in (topo_row, feat_row):
        if int(row.max().item() if row.numel() else 0) > MAX_HOTNESS:
            raise OverflowError("hotness counts exceed the packed owner all-reduce range")
        totals = row.clone()
        dist.all_reduce(totals, op=dist.ReduceOp.SUM, group=group)
        packed = (row << OWNER_BITS) | ((1 << OWNER_BITS) - 1 - local_rank)
        dist.all_reduce(packed, op=dist.ReduceOp.MAX, group=group)
        owner = ((1 << OWNER_BITS) - 1 - (packed & ((1 << OWNER_BITS) - 1))).to(torch.int32)
        out += [totals, owner]
    return tuple(out)


def candidate_orders_from_rows(topo_row: torch.Tensor, feat_row: torch.Tensor, local_rank: int, clique_size: int,
                               clique_id: int = 0, group=None):
    """build_candidate_orders (planner.py:48-67) when each rank holds its own hotness
    row: merge with two all-reduces, then rank locally (every rank computes the same
    deterministic order, so no broadcast is needed)."""
    from .planner import CandidateOrders, device_descending_order, device_distribute

    tt, to, ft, fo = merge_hotness(topo_row, feat_row, local_rank, group)
    dev = {}
    res = {}
    for kind, totals, owner in (("topo", tt, to), ("feat", ft, fo)):
        totals, owner = totals.cuda(), owner.cuda()
        order = device_descending_order(totals)
        queues = device_distribute(order, order.numel(), owner, clique_size)
        dev.update({f"{kind}_totals": totals, f"{kind}_order": order, f"{kind}_owner": owner})
        res[kind] = (totals.cpu().numpy(), order.cpu().numpy(), owner.cpu().numpy(),
                     tuple(q.cpu().numpy() for q in queues))
    return CandidateOrders(clique_id, res["topo"][0], res["feat"][0], res["topo"][1], res["feat"][1],
                           res["topo"][2], res["feat"][2], res["topo"][3], res["feat"][3], _device=dev)


def ipc_export(t: torch.Tensor) -> bytes:
    """64-byte CUDA IPC handle of the cudaMalloc allocation holding tensor t, plus t's
    byte offset from that allocation's base (torch's caching allocator places many
    tensors inside one allocation; cudaIpcOpenMemHandle maps the allocation base)."""
    import ctypes

    lib = _lib.lib()
    buf = ctypes_buffer()
    off = ctypes.c_uint64(0)
    _lib.check(lib.gc_ipc_export(t.data_ptr(), buf, ctypes.byref(off)), "ipc_export")
    return bytes(buf.raw[:64]) + int(off.value).to_bytes(8, "little")


def ipc_import(blob: bytes) -> int:
    """Map a peer's exported allocation; returns the device address of the tensor."""
    import ctypes

    lib = _lib.lib()
    ptr = ctypes.c_void_p()
    _lib.check(lib.gc_ipc_import(blob[:64], ctypes.byref(ptr)), "ipc_import")
    return int(ptr.value) + int.from_bytes(blob[64:72], "little")


def ctypes_buffer():
    import ctypes

    return ctypes.create_string_buffer(64)


def exchange_addresses(local: list, rank: int, world: int, group=None, export=None, import_=None) -> list[list]:
    """All-gather per-rank exported handles of `local` (a list of tensors) and map the
    peers'. Returns addr[g][i]: device address of rank g's i-th tensor as seen from this
    rank (own tensors are returned as-is). export/import_ default to CUDA IPC; tests
    inject stand-ins to exercise the exchange logic on CPU."""
    if world == 1:
        return [list(local)]
    export = export or ipc_export
    import_ = import_ or ipc_import
    mine = [export(t) for t in local]
    everyone: list = [None] * world
    dist.all_gather_object(everyone, mine, group=group)
    out = []
    for g in range(world):
        if g == rank:
            out.append(list(local))
        else:
            out.append([import_(b) for b in everyone[g]])
    return out


def max_over_ranks(value: float, group=None) -> float:
    """Max of a host scalar over ranks (device-timed results, never wall clock)."""
    if not dist.is_initialized():
        return value
    backend = dist.get_backend(group)
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: int, group=None) -> int:
    if not dist.is_initialized():
        return value
    backend = dist.get_backend(group)
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.int64, device=dev)
    dist.all_reduce(t, group=group)
    return int(t.item())


def rows_numpy_merge_reference(rows: np.ndarray):
    """What merge_hotness must equal: column sums and np.argmax owners (planner.py:50-55)."""
    return rows.sum(axis=0), np.argmax(rows, axis=0).astype(np.int32)
