"""ctypes binding of libgnncache_b200.so (include/gnncache_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``. There is no CPU
fallback for the sampling/gather path: if the library or a CUDA device is missing,
every entry point raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

LIB_NAME = "libgnncache_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

GC_OK = 0
GC_ERR_VALUE = -1
GC_ERR_OVERFLOW = -2
GC_ERR_CUDA = -3
GC_ERR_UNSUPPORTED = -4
GC_ERR_ASSERT = -5
GC_MAX_PEERS = 8
GC_OPT_EXACT_SELECTION = 1
GC_OPT_DEFER_CTAS = 2
GC_OPT_GATHER_CTAS_PER_SM = 3
GC_OPT_UNIQUE_BATCH_CTAS = 4
GC_OPT_DEFER_ORDER = 5
GC_OPT_DEFER_ROWS = 6
GC_TIER_HOST = 0xFFFFFFFF

_c_u64p = ctypes.c_void_p  # every device pointer crosses as an opaque address


class GcCsr(ctypes.Structure):
    _fields_ = [
        ("num_vertices", ctypes.c_int64),
        ("num_edges", ctypes.c_int64),
        ("row_offsets", ctypes.c_void_p),
        ("col_indices", ctypes.c_void_p),
    ]


class GcTopology(ctypes.Structure):
    _fields_ = [
        ("full", GcCsr),
        ("location", ctypes.c_void_p),
        ("slab_offsets", ctypes.c_void_p * 8),
        ("slab_cols", ctypes.c_void_p * 8),
        ("self_rank", ctypes.c_uint32),
        ("full_on_host", ctypes.c_uint32),
        ("tier_reads", ctypes.c_void_p),
    ]


class GcVisited(ctypes.Structure):
    _fields_ = [
        ("bitmap", ctypes.c_void_p),
        ("words", ctypes.c_uint64),
        ("summary", ctypes.c_void_p),
        ("summary_words", ctypes.c_uint64),
    ]


class GcHotness(ctypes.Structure):
    _fields_ = [
        ("topo_reads", ctypes.c_void_p),
        ("edge_traversals", ctypes.c_void_p),
        ("feat_lookups", ctypes.c_void_p),
        ("txn_total", ctypes.c_void_p),
        ("cache_line_bytes", ctypes.c_uint32),
        ("uint32_bytes", ctypes.c_uint32),
    ]


class GcFeatureStore(ctypes.Structure):
    _fields_ = [
        ("row_bytes", ctypes.c_uint32),
        ("self_rank", ctypes.c_uint32),
        ("num_ranks", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("location", ctypes.c_void_p),
        ("slabs", ctypes.c_void_p * GC_MAX_PEERS),
        ("host_rows", ctypes.c_void_p),
    ]


GC_TREE_MAX_LEVELS = 8


class GcTreeSrc(ctypes.Structure):
    _fields_ = [
        ("hops", ctypes.c_int32),
        ("counts", ctypes.c_void_p),
        ("counts_stride", ctypes.c_int64),
        ("local", ctypes.c_void_p * GC_TREE_MAX_LEVELS),
        ("local_stride", ctypes.c_int64 * GC_TREE_MAX_LEVELS),
        ("offsets", ctypes.c_void_p * GC_TREE_MAX_LEVELS),
        ("offsets_stride", ctypes.c_int64 * GC_TREE_MAX_LEVELS),
        ("seeds", ctypes.c_void_p),
        ("seeds_stride", ctypes.c_int64),
        ("labels", ctypes.c_void_p),
        ("caps", ctypes.c_int64 * GC_TREE_MAX_LEVELS),
        ("local_bits", ctypes.c_int32),
    ]


V = ctypes.c_void_p
I32 = ctypes.c_int32
U32 = ctypes.c_uint32
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
SZ = ctypes.c_size_t
D = ctypes.c_double

# name -> (restype, argtypes); must cover every symbol include/gnncache_b200.h declares
SIGNATURES = {
    "gc_abi_version": (ctypes.c_int, []),
    "gc_last_error": (ctypes.c_char_p, []),
    "gc_current_device": (ctypes.c_int, []),
    "gc_set_option": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "gc_mix64": (ctypes.c_int, [V, V, I64, V]),
    "gc_hash_counters": (ctypes.c_int, [U64, V, V, I64, V]),
    "gc_hash_pairs": (ctypes.c_int, [U64, V, V, V, I64, V]),
    "gc_permutation_temp_bytes": (SZ, [I64]),
    "gc_permutation": (ctypes.c_int, [U64, I64, V, V, V, SZ, V]),
    "gc_permutation_dkey": (ctypes.c_int, [V, I64, V, V, V, SZ, V]),
    "gc_hop_expand_temp_bytes": (SZ, [U32, U32]),
    "gc_hop_expand": (
        ctypes.c_int,
        [ctypes.POINTER(GcTopology), V, U64, V, U32, U32, V, U32, V, U64, V, U64, V, ctypes.POINTER(GcVisited),
         ctypes.c_int, ctypes.POINTER(GcHotness), V, SZ, V],
    ),
    "gc_csr_extract": (ctypes.c_int, [ctypes.POINTER(GcCsr), V, I64, V, V, V]),
    "gc_bitmap_words": (U64, [I64]),
    "gc_summary_words": (U64, [I64]),
    "gc_unique_temp_bytes": (SZ, [U32, ctypes.POINTER(GcVisited)]),
    "gc_unique_compact": (ctypes.c_int, [ctypes.POINTER(GcVisited), U32, V, U64, V, V, V, ctypes.c_int, V, SZ, V]),
    "gc_unique_compact_launches": (ctypes.c_int, [U32, ctypes.POINTER(GcVisited)]),
    "gc_relabel": (ctypes.c_int, [V, U64, V, U32, U32, V, U64, V, V]),
    "gc_relabel16": (ctypes.c_int, [V, U64, V, U32, U32, V, U64, V, V]),
    "gc_mark_visited": (ctypes.c_int, [V, U64, V, U32, U32, ctypes.POINTER(GcVisited), V]),
    "gc_synth_features": (ctypes.c_int, [U64, U64, U32, V, V]),
    "gc_bitmap_clear": (ctypes.c_int, [ctypes.POINTER(GcVisited), U32, V, U64, V, U32, V]),
    "gc_gather": (ctypes.c_int, [ctypes.POINTER(GcFeatureStore), V, U64, V, U32, U32, V, U64, V, V]),
    "gc_scatter_add": (ctypes.c_int, [V, V, I64, V, V]),
    "gc_segment_mean_gather": (ctypes.c_int, [V, ctypes.c_int, V, V, I64, V, V]),
    "gc_tree_stage": (ctypes.c_int, [ctypes.POINTER(GcTreeSrc), V, V, V, V, V, V, V]),
    "gc_tree_aggregate": (ctypes.c_int, [V, ctypes.c_int, I64, ctypes.c_int, V, V, V, I64, ctypes.c_int, V,
                                         ctypes.c_int, I64, V, I64, V]),
    "gc_tree_aggregate_backward": (ctypes.c_int, [V, ctypes.c_int, I64, ctypes.c_int, ctypes.c_int, V, V, I64, I64,
                                                  V, I64, V, I64, ctypes.c_int, ctypes.POINTER(I64), V, V]),
    "gc_colsum_argmax": (ctypes.c_int, [V, U32, I64, V, V, V]),
    "gc_descending_order_temp_bytes": (SZ, [I64]),
    "gc_descending_order": (ctypes.c_int, [V, I64, V, V, SZ, V]),
    "gc_order_scan_temp_bytes": (SZ, [I64]),
    "gc_topo_prefix_bytes": (ctypes.c_int, [V, V, I64, U32, U32, V, V, SZ, V]),
    "gc_hot_prefix": (ctypes.c_int, [V, V, I64, V, V, SZ, V]),
    "gc_searchsorted_right": (ctypes.c_int, [V, I64, V, I32, V, V]),
    "gc_distribute_prefix_temp_bytes": (SZ, [I64, U32]),
    "gc_distribute_prefix": (ctypes.c_int, [V, I64, V, U32, V, V, V, SZ, V]),
    "gc_mark_holders": (ctypes.c_int, [V, I64, U32, V, V]),
    "gc_tier_account": (ctypes.c_int, [V, I64, V, V, V, V, U32, U32, U32, U32, U32, V, V]),
    "gc_host_register": (ctypes.c_int, [V, SZ, ctypes.POINTER(ctypes.c_void_p)]),
    "gc_gather_defer_bytes": (U64, [U32, U32]),
    "gc_gather_deferred": (ctypes.c_int,
                           [ctypes.POINTER(GcFeatureStore), V, U64, V, U32, U32, V, U64, V, V, U64, V, V]),
    "gc_host_unregister": (ctypes.c_int, [V]),
    "gc_copy_d2h_mapped": (ctypes.c_int, [V, V, U64, V]),
    "gc_tree_head_work_floats": (SZ, [I64, ctypes.c_int, ctypes.c_int]),
    "gc_tree_head": (ctypes.c_int, [V, ctypes.c_int, I64, ctypes.c_int, I64, V, V, ctypes.c_int, V, V, V, V, V, V,
                                    I64, V, SZ, V]),
    "gc_pack_segments": (ctypes.c_int, [V, U64, U64, V, U32, U64, ctypes.c_int, V, V]),
    "gc_host_alloc_numa": (ctypes.c_int, [SZ, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(SZ)]),
    "gc_host_free_numa": (ctypes.c_int, [V, SZ]),
    "gc_synth_zipf_targets": (ctypes.c_int, [U64, U64, U64, U64, V, U64, U64, U64, U64, V, V]),
    "gc_ipc_export": (ctypes.c_int, [V, ctypes.c_char_p, ctypes.POINTER(U64)]),
    "gc_ipc_import": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "gc_ipc_close": (ctypes.c_int, [V]),
    "gc_enable_peer": (ctypes.c_int, [ctypes.c_int]),
    "gc_partition_ldg": (ctypes.c_int, [V, V, U64, U64, V, U32, I64, ctypes.c_int, V, V]),
}

_LIB = None


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing; there is no CPU fallback."""


def load_library(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load the shared library and bind every header symbol (no GPU needed)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    # GC_LIB_PATH: load an experimental build (tools/build_variant.py) instead
    p = Path(path) if path is not None else Path(os.environ.get("GC_LIB_PATH", LIB_PATH))
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.gc_abi_version() != 1:
        raise NativeUnavailable("libgnncache_b200.so ABI version mismatch")
    if path is None:
        _LIB = lib
    return lib


def lib() -> ctypes.CDLL:
    """The library, with a CUDA device required (every compute call goes through here)."""
    if not torch.cuda.is_available():
        raise NativeUnavailable("a CUDA device is required: the B200 path has no CPU fallback")
    return load_library()


def check(status: int, what: str = "") -> None:
    if status == GC_OK:
        return
    msg = (_LIB.gc_last_error() or b"").decode(errors="replace") if _LIB else ""
    text = f"{what}: {msg}" if what else msg
    if status == GC_ERR_VALUE:
        raise ValueError(text)
    if status == GC_ERR_OVERFLOW:
        raise OverflowError(text)
    if status == GC_ERR_ASSERT:
        raise AssertionError(text)
    if status == GC_ERR_UNSUPPORTED:
        raise NotImplementedError(text)
    raise RuntimeError(text)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def u64(x: int) -> int:
    return int(x) & 0xFFFFFFFFFFFFFFFF
