"""Mini-batch L-hop sampling and presampling hotness on the B200 (sampling.py of the reference).

Same public API, dataclasses, counting rules and exceptions as the reference; every
array operation of the path runs in libgnncache_b200.so:

  K1 local shuffle      KeyedRng.permutation -> gc_permutation (stable radix sort)
  K2 hop expansion      _expand_frontier     -> gc_hop_expand (one launch per hop per window of batches)
  K3 dedup (+relabel)   distinct_vertices    -> visited bitmaps + gc_unique_compact
  K5 hotness            bincount x3          -> counters fused into K2/K3

`WindowSampler` is the engine: it samples a window of W batches with one launch per
hop, keeping frontier sizes on the device so no host round trip happens between
hops. `sample_batch`, `run_sampling_epoch` and `run_presampling` are thin host
drivers over it.
"""

from __future__ import annotations

import math
import struct
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph
from .hardware import CliqueLayout, HardwareSpec
from .rng import GOLDEN, MASK64, ROLE_SAMPLE, ROLE_SHUFFLE, KeyedRng, mix64


@dataclass(frozen=True)
class SamplingConfig:
    """Fanouts, batch size, presampling epochs, seed (sampling.py:28-48)."""

    fanouts: tuple[int, ...]
    batch_size: int
    presample_epochs: int = 1
    seed: int = 0
    num_hops: int | None = None

    def __post_init__(self):
        fanouts = tuple(int(f) for f in self.fanouts)
        object.__setattr__(self, "fanouts", fanouts)
        hops = len(fanouts) if self.num_hops is None else self.num_hops
        object.__setattr__(self, "num_hops", hops)
        if hops != len(fanouts):
            raise ValueError("num_hops must equal len(fanouts)")
        if any(f < 1 for f in fanouts):
            raise ValueError("fanouts must all be >= 1")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.presample_epochs < 0:
            raise ValueError("presample_epochs must be >= 0")


@dataclass(frozen=True)
class HopExpansion:
    """One hop: ragged source -> sampled-neighbour lists (sampling.py:51-66)."""

    sources: np.ndarray
    offsets: np.ndarray
    neighbors: np.ndarray

    def pairs(self):
        for i, src in enumerate(self.sources):
            yield int(src), self.neighbors[self.offsets[i] : self.offsets[i + 1]]

    @property
    def sampled_counts(self) -> np.ndarray:
        return np.diff(self.offsets)


@dataclass(frozen=True)
class BatchSample:
    """Seeds plus per-hop expansions (sampling.py:69-75)."""

    seeds: np.ndarray
    hops: tuple[HopExpansion, ...]

    def distinct_vertices(self) -> np.ndarray:
        """Sorted distinct ids of seeds ∪ all hop neighbours, computed on the device
        (bitmap dedup) — or the result the device produced while sampling."""
        cached = self.__dict__.get("_distinct")
        if cached is not None:
            return cached.copy()
        parts = [np.asarray(self.seeds, dtype=np.int64)] + [np.asarray(h.neighbors, dtype=np.int64) for h in self.hops]
        ids = np.concatenate(parts)
        if len(ids) == 0:
            return np.empty(0, dtype=np.int64)
        if ids.min() < 0 or ids.max() > 0xFFFFFFFF:
            raise ValueError("vertex ids must lie in [0, 2^32)")
        return device_unique(ids, int(ids.max()) + 1)


# ----------------------------------------------------------------------------- keys


def _mix64_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    x ^= x >> np.uint64(30)
    x *= np.uint64(0xBF58476D1CE4E5B9)
    x ^= x >> np.uint64(27)
    x *= np.uint64(0x94D049BB133111EB)
    x ^= x >> np.uint64(31)
    return x


def batch_hop_keys(gpu_stream: KeyedRng, first_batch: int, num_batches: int, num_hops: int) -> np.ndarray:
    """keys[b, h] = gpu_stream.derive(ROLE_SAMPLE, first_batch + b).derive(h).key
    (sampling.py:234 and :135), vectorised over batches. uint64 [num_batches, num_hops]."""
    with np.errstate(over="ignore"):
        k_role = np.uint64(mix64(gpu_stream.key ^ mix64((ROLE_SAMPLE + GOLDEN) & MASK64)))
        b = np.arange(first_batch, first_batch + num_batches, dtype=np.uint64)
        k_batch = _mix64_np(k_role ^ _mix64_np(b + np.uint64(GOLDEN)))
        out = np.empty((num_batches, num_hops), dtype=np.uint64)
        for h in range(num_hops):
            out[:, h] = _mix64_np(k_batch ^ np.uint64(mix64((h + GOLDEN) & MASK64)))
    return out


# --------------------------------------------------------------------------- engine


class DeviceHotness:
    """GpuTrace counters of one GPU resident in HBM (u64)."""

    def __init__(self, n: int, spec: HardwareSpec | None = None):
        self.topo_reads = torch.zeros(n, dtype=torch.int64, device="cuda")
        self.edge_traversals = torch.zeros(n, dtype=torch.int64, device="cuda")
        self.feat_lookups = torch.zeros(n, dtype=torch.int64, device="cuda")
        self.txn_total = torch.zeros(1, dtype=torch.int64, device="cuda")
        cls = spec.cache_line_bytes if spec else 64
        u32 = spec.uint32_bytes if spec else 4
        self.c_struct = _lib.GcHotness(
            self.topo_reads.data_ptr(),
            self.edge_traversals.data_ptr(),
            self.feat_lookups.data_ptr(),
            self.txn_total.data_ptr(),
            cls,
            u32,
        )


class WindowSampler:
    """Samples W mini-batches per launch: hop expansion, dedup, relabel and gather.

    Device layout (per batch b, fixed strides so the window is one launch per stage):
      seeds     u32 [W, B]                 counts[0] u32 [W]
      hop h     offsets u32 [W, cap_h + 1], neighbours u32 [W, cap_{h+1}], counts[h+1]
      bitmap    u32 [W, words]              visited set of the batch (zero between windows)
      unique    u32 [W, ucap]               sorted distinct ids, ucount u32 [W]
    with cap_0 = B and cap_{h+1} = cap_h * fanout_h (frontiers are not deduplicated
    between hops, sampling.py:123-125).
    """

    # above this many vertices the visited sets carry a block summary (sparse compaction)
    SPARSE_VISITED_MIN_VERTICES = 1 << 22

    def __init__(self, graph: CsrGraph, fanouts, batch_size: int, window: int, *, placement: str = "hbm",
                 relabel: bool = False, unique_cap: int | None = None, topology=None,
                 sparse_visited: bool | None = None):
        self.lib = _lib.lib()
        self.graph = graph
        # topology: a cache.TopologyStore (tiered lists) or the plain CSR in `placement`
        self.topology = topology
        self.topo_struct = topology.c_struct if topology is not None else graph.device(placement).topology
        self.n = graph.num_vertices
        self.fanouts = tuple(int(f) for f in fanouts)
        self.H = len(self.fanouts)
        self.B = int(batch_size)
        self.W = int(window)
        if not 1 <= self.W <= MAX_WINDOW:
            raise ValueError(f"window must be in [1, {MAX_WINDOW}] batches")
        self.relabel = relabel
        caps = [self.B]
        for f in self.fanouts:
            if caps[-1] * f >= 1 << 32:
                raise ValueError("per-batch hop output must stay below 2^32 entries")
            caps.append(caps[-1] * f)
        self.caps = caps
        W, dev = self.W, "cuda"
        i32 = torch.int32
        self.seeds = torch.zeros((W, self.B), dtype=i32, device=dev)
        self.counts = torch.zeros((self.H + 1, W), dtype=i32, device=dev)
        self.offsets = [torch.empty((W, caps[h] + 1), dtype=i32, device=dev) for h in range(self.H)]
        self.nbrs = [torch.empty((W, max(caps[h + 1], 1)), dtype=i32, device=dev) for h in range(self.H)]
        self.keys = torch.zeros((self.H, W), dtype=torch.int64, device=dev)
        self.words = int(self.lib.gc_bitmap_words(self.n))
        self.bitmap = torch.zeros((W, self.words), dtype=i32, device=dev)
        if sparse_visited is None:
            sparse_visited = self.n >= self.SPARSE_VISITED_MIN_VERTICES
        self.swords = int(self.lib.gc_summary_words(self.n)) if sparse_visited else 0
        self.summary = torch.zeros((W, self.swords), dtype=i32, device=dev) if sparse_visited else None
        self.visited = _lib.GcVisited(self.bitmap.data_ptr(), self.words, _lib.ptr(self.summary), self.swords)
        bound = min(self.n, sum(caps))
        self.ucap = max(1, bound if unique_cap is None else min(bound, int(unique_cap)))
        # capped unique buffers can overflow: the compaction writes at most ucap ids and
        # still reports the true count, whose running maximum is kept on the device
        # (no sync per window) and checked by check_capacity()
        self.peak_ucount = torch.zeros((), dtype=i32, device=dev) if self.ucap < bound else None
        self.unique = torch.empty((W, self.ucap), dtype=i32, device=dev)
        self.ucount = torch.zeros(W, dtype=i32, device=dev)
        # relabel rank table: {exclusive popcount prefix, bitmap word} per word
        self.rank = torch.empty((W, 2 * self.words), dtype=i32, device=dev) if relabel else None
        # local ids as u16 (held in int16 tensors) when no batch can have more than 65536
        # distinct vertices: a quarter less traffic for the relabel pass and half the bytes
        # its consumers read; decode with local_ids()
        self.local_bits = 16 if relabel and self.ucap <= 1 << 16 else 32
        ldt = torch.int16 if self.local_bits == 16 else i32
        self.local_seeds = torch.empty((W, self.B), dtype=ldt, device=dev) if relabel else None
        self.local_nbrs = [torch.empty(t.shape, dtype=ldt, device=dev) for t in self.nbrs] if relabel else None
        hop_tmp = max([self.lib.gc_hop_expand_temp_bytes(W, caps[h]) for h in range(self.H)] + [256])
        self.hop_tmp = torch.empty(hop_tmp, dtype=torch.uint8, device=dev)
        uq_tmp = self.lib.gc_unique_temp_bytes(W, self.visited)
        self.uq_tmp = torch.empty(uq_tmp, dtype=torch.uint8, device=dev)
        self.active = 0

    # ---- inputs
    def load(self, seeds_flat: torch.Tensor, counts: np.ndarray, keys: np.ndarray) -> None:
        """seeds_flat: int32 CUDA tensor holding the window's seeds batch after batch
        (batch b = seeds_flat[b*B : b*B + counts[b]]); keys: uint64 [nb, H]."""
        nb = len(counts)
        if nb > self.W:
            raise ValueError("more batches than the window holds")
        self.active = nb
        total = int(counts.sum())
        flat = self.seeds.view(-1)
        flat[:total].copy_(seeds_flat[:total], non_blocking=True)
        cnt = torch.from_numpy(np.asarray(counts, dtype=np.int32))
        self.counts[0, :nb].copy_(cnt, non_blocking=True)
        if self.H:
            kt = torch.from_numpy(np.ascontiguousarray(keys.T).view(np.int64))
            self.keys[:, :nb].copy_(kt, non_blocking=True)

    # ---- stages
    def expand(self, hot: DeviceHotness | None = None, stream=None, timer=None) -> None:
        nb = self.active
        s = _lib.stream_handle(stream)
        hp = hot.c_struct if hot is not None else None
        for h, f in enumerate(self.fanouts):
            end = timer.start(f"hop_expand.h{h}") if timer is not None else None
            front = self.seeds if h == 0 else self.nbrs[h - 1]
            _lib.check(
                self.lib.gc_hop_expand(
                    self.topo_struct, front.data_ptr(), front.shape[1], self.counts[h].data_ptr(), self.caps[h], f,
                    self.keys[h].data_ptr(), nb, self.offsets[h].data_ptr(), self.offsets[h].shape[1],
                    self.nbrs[h].data_ptr(), self.nbrs[h].shape[1], self.counts[h + 1].data_ptr(),
                    self.visited, 1 if h == 0 else 0, hp,
                    self.hop_tmp.data_ptr(), self.hop_tmp.numel(), s,
                ),
                "hop_expand",
            )
            if end is not None:
                end.record()
        if self.H == 0:
            _lib.check(
                self.lib.gc_mark_visited(self.seeds.data_ptr(), self.B, self.counts[0].data_ptr(), self.B, nb,
                                         self.visited, s),
                "mark_visited",
            )

    def dedup(self, hot: DeviceHotness | None = None, stream=None, relabel_stream=None) -> None:
        """Sorted unique ids per batch; the visited bitmap is cleared as it is consumed
        (relabel reads the interleaved rank table instead). relabel_stream: run the
        relabel launches there (ordered after the compaction) so they overlap whatever
        the caller enqueues next on `stream`; the caller joins that stream."""
        s = _lib.stream_handle(stream)
        _lib.check(
            self.lib.gc_unique_compact(
                self.visited, self.active, self.unique.data_ptr(), self.ucap,
                self.ucount.data_ptr(), _lib.ptr(self.rank), hot.feat_lookups.data_ptr() if hot else None,
                1, self.uq_tmp.data_ptr(), self.uq_tmp.numel(), s,
            ),
            "unique_compact",
        )
        if self.peak_ucount is not None and self.active:
            with torch.cuda.stream(stream) if stream is not None else _nullcontext():
                torch.maximum(self.peak_ucount, self.ucount[: self.active].amax(), out=self.peak_ucount)
        if self.relabel:
            if relabel_stream is not None:
                ready = torch.cuda.Event()
                ready.record(stream if stream is not None else torch.cuda.current_stream())
                relabel_stream.wait_event(ready)
                s = _lib.stream_handle(relabel_stream)
            arrays = [(self.seeds, self.counts[0], self.local_seeds, self.B)] + [
                (self.nbrs[h], self.counts[h + 1], self.local_nbrs[h], self.caps[h + 1]) for h in range(self.H)
            ]
            fn = self.lib.gc_relabel16 if self.local_bits == 16 else self.lib.gc_relabel
            for ids, cnt, loc, cap in arrays:
                _lib.check(fn(ids.data_ptr(), ids.shape[1], cnt.data_ptr(), cap, self.active, self.rank.data_ptr(),
                              self.words, loc.data_ptr(), s), "relabel")

    def check_capacity(self, reset: bool = False) -> int:
        """Largest distinct count of any batch since the last reset (one sync); raises
        OverflowError when it exceeded the unique-row capacity, i.e. some batch's
        distinct ids (and gathered rows) were truncated."""
        if self.peak_ucount is None:
            return -1
        peak = int(self.peak_ucount.item())
        if reset:
            self.peak_ucount.zero_()
        if peak > self.ucap:
            raise OverflowError(f"a batch has {peak} distinct vertices but the unique/gather capacity is "
                                f"{self.ucap}: raise feat_rows_cap")
        return peak

    def run(self, hot: DeviceHotness | None = None, stream=None) -> None:
        self.expand(hot, stream)
        self.dedup(hot, stream=stream)

    # ---- host views (API drivers / tests)
    def batch_to_host(self, b: int) -> BatchSample:
        counts = self.counts[:, b].cpu().numpy().astype(np.int64)
        seeds = self.seeds[b, : counts[0]].cpu().numpy().view(np.uint32).astype(np.int64)
        hops = []
        front = seeds
        for h in range(self.H):
            f = int(counts[h])
            if f == 0:
                empty = np.empty(0, dtype=np.int64)
                hops.append(HopExpansion(empty, np.zeros(1, dtype=np.int64), empty))
                continue
            offs = self.offsets[h][b, : f + 1].cpu().numpy().view(np.uint32).astype(np.int64)
            nb = self.nbrs[h][b, : counts[h + 1]].cpu().numpy().view(np.uint32).astype(np.int64)
            hops.append(HopExpansion(front, offs, nb))
            front = nb
        out = BatchSample(seeds, tuple(hops))
        u = int(self.ucount[b].item())
        object.__setattr__(out, "_distinct", self.unique[b, :u].cpu().numpy().view(np.uint32).astype(np.int64))
        return out


class _nullcontext:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def check_seed_pool(pool, num_vertices: int) -> None:
    """sample_batch's seed check (sampling.py:128-131) for a whole pool: ValueError
    before any id reaches a kernel (numpy pools on the host; device pools with one
    min/max reduction)."""
    if isinstance(pool, torch.Tensor):
        if pool.numel() == 0:
            return
        lo, hi = torch.aminmax(pool)
        lo, hi = int(lo.item()), int(hi.item())
    else:
        arr = np.asarray(pool)
        if arr.size == 0:
            return
        lo, hi = int(arr.min()), int(arr.max())
    if lo < 0 or hi >= num_vertices:
        raise ValueError("invalid seed vertex id")


def device_unique(ids: np.ndarray, n: int) -> np.ndarray:
    """np.unique of one id list through the bitmap dedup kernels."""
    lib = _lib.lib()
    words = int(lib.gc_bitmap_words(n))
    swords = int(lib.gc_summary_words(n))
    d_ids = torch.from_numpy(ids.astype(np.uint32).view(np.int32)).cuda()
    cnt = torch.tensor([len(ids)], dtype=torch.int32, device="cuda")
    bm = torch.zeros(words, dtype=torch.int32, device="cuda")
    sm = torch.zeros(swords, dtype=torch.int32, device="cuda")
    vis = _lib.GcVisited(bm.data_ptr(), words, sm.data_ptr(), swords)
    s = _lib.stream_handle()
    _lib.check(lib.gc_mark_visited(d_ids.data_ptr(), len(ids), cnt.data_ptr(), len(ids), 1, vis, s))
    cap = min(n, len(ids))
    uniq = torch.empty(max(cap, 1), dtype=torch.int32, device="cuda")
    ucnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    tmp = torch.empty(lib.gc_unique_temp_bytes(1, vis), dtype=torch.uint8, device="cuda")
    _lib.check(lib.gc_unique_compact(vis, 1, uniq.data_ptr(), cap, ucnt.data_ptr(), None, None, 1,
                                     tmp.data_ptr(), tmp.numel(), s))
    return uniq[: int(ucnt.item())].cpu().numpy().view(np.uint32).astype(np.int64)


_SINGLE: dict = {}


def _single_sampler(graph: CsrGraph, fanouts: tuple[int, ...], nseeds: int) -> WindowSampler:
    cap = 1 << max(0, (nseeds - 1).bit_length())
    key = (id(graph), fanouts, cap, torch.cuda.current_device())
    ent = _SINGLE.get(key)
    if ent is None or ent[0] is not graph:
        if len(_SINGLE) > 16:
            _SINGLE.clear()
        ent = (graph, WindowSampler(graph, fanouts, cap, 1))
        _SINGLE[key] = ent
    return ent[1]


def sample_batch(graph: CsrGraph, seeds, cfg: SamplingConfig, stream: KeyedRng) -> BatchSample:
    """L-hop uniform neighbour sampling of one mini-batch (sampling.py:120-143);
    hop h uses stream.derive(h), a vertex sampled twice is expanded twice."""
    seeds = np.asarray(seeds, dtype=np.int64)
    if len(seeds) == 0:
        raise ValueError("seeds must be non-empty")
    if seeds.min() < 0 or seeds.max() >= graph.num_vertices:
        raise ValueError("invalid seed vertex id")
    sampler = _single_sampler(graph, cfg.fanouts, len(seeds))
    keys = np.array([[stream.derive(h).key for h in range(len(cfg.fanouts))]], dtype=np.uint64).reshape(1, -1)
    dev = torch.from_numpy(seeds.astype(np.uint32).view(np.int32)).cuda()
    sampler.load(dev, np.array([len(seeds)]), keys)
    sampler.run()
    return sampler.batch_to_host(0)


# ------------------------------------------------------------------------ hotness


@dataclass
class HotnessMatrices:
    """Per-clique hotness rows plus the sampling transaction total (sampling.py:146-161)."""

    clique_id: int
    topo_hotness: np.ndarray
    feat_hotness: np.ndarray
    sampling_txn_total: int = 0

    @property
    def clique_size(self) -> int:
        return self.topo_hotness.shape[0]

    @property
    def num_vertices(self) -> int:
        return self.topo_hotness.shape[1]


def accumulate_hotness(batch: BatchSample, gpu_row: int, hotness: HotnessMatrices) -> HotnessMatrices:
    """Fold one batch into a GPU's rows (sampling.py:164-174), as device scatter-adds."""
    lib = _lib.lib()
    n = hotness.num_vertices
    s = _lib.stream_handle()
    topo = torch.zeros(n, dtype=torch.int64, device="cuda")
    for hop in batch.hops:
        if len(hop.sources) == 0:
            continue
        src = torch.from_numpy(np.asarray(hop.sources).astype(np.uint32).view(np.int32)).cuda()
        w = torch.from_numpy(hop.sampled_counts.astype(np.uint32).view(np.int32)).cuda()
        _lib.check(lib.gc_scatter_add(src.data_ptr(), w.data_ptr(), src.numel(), topo.data_ptr(), s), "scatter_add")
    feat = torch.zeros(n, dtype=torch.int64, device="cuda")
    d = batch.distinct_vertices()
    if len(d):
        ids = torch.from_numpy(d.astype(np.uint32).view(np.int32)).cuda()
        _lib.check(lib.gc_scatter_add(ids.data_ptr(), None, ids.numel(), feat.data_ptr(), s), "scatter_add")
    hotness.topo_hotness[gpu_row] += topo.cpu().numpy()
    hotness.feat_hotness[gpu_row] += feat.cpu().numpy()
    return hotness


def topology_access_cost(graph: CsrGraph, v: int, spec: HardwareSpec) -> int:
    """t(v) = 1 + ceil(nc(v) * uint32_bytes / CLS) (sampling.py:177-180)."""
    cls = spec.cache_line_bytes
    return 1 + (graph.out_degree(v) * spec.uint32_bytes + cls - 1) // cls


def transaction_cost_table(graph: CsrGraph, spec: HardwareSpec) -> np.ndarray:
    """t(v) for all v, int64 (sampling.py:183-187)."""
    cls = spec.cache_line_bytes
    return 1 + (graph.out_degrees * spec.uint32_bytes + cls - 1) // cls


@dataclass
class GpuTrace:
    """Access counts of one GPU over one epoch (sampling.py:190-197)."""

    topo_reads: np.ndarray
    feat_lookups: np.ndarray
    edge_traversals: np.ndarray
    num_batches: int = 0


MAX_WINDOW = 65535  # batches per window: the hop/pack kernels put the batch in grid.y


def local_ids(t: torch.Tensor) -> torch.Tensor:
    """WindowSampler local ids as int64, whatever their storage (u16 held in int16, or int32)."""
    if t.dtype == torch.int16:
        return t.to(torch.int32).bitwise_and_(0xFFFF).long()
    return t.long()


def _window_for(sampler_caps: list[int], words: int, num_batches: int, budget_bytes: int = 2 << 30) -> int:
    per_batch = 4 * (2 * sum(sampler_caps) + len(sampler_caps) + 2 * words) + 4 * min(sum(sampler_caps), 1 << 30)
    # <= 65535: the batch index is a launch's grid.y
    return max(1, min(num_batches, budget_bytes // max(per_batch, 1), MAX_WINDOW))


class EpochRunner:
    """Local shuffle + windowed sampling of one GPU's pool for one epoch (sampling.py:224-243)."""

    def __init__(self, graph: CsrGraph, cfg: SamplingConfig, max_pool: int, placement: str = "hbm",
                 sparse_visited: bool | None = None):
        self.graph = graph
        self.cfg = cfg
        lib = _lib.lib()
        caps = [cfg.batch_size]
        for f in cfg.fanouts:
            caps.append(caps[-1] * f)
        words = int(lib.gc_bitmap_words(graph.num_vertices))
        nb = max(1, math.ceil(max_pool / cfg.batch_size))
        self.window = _window_for(caps, words, nb)
        self.sampler = WindowSampler(graph, cfg.fanouts, cfg.batch_size, self.window, placement=placement,
                                     sparse_visited=sparse_visited)

    def run(self, pool: np.ndarray, gpu_stream: KeyedRng, hot: DeviceHotness) -> int:
        B = self.cfg.batch_size
        L = len(pool)
        check_seed_pool(pool, self.graph.num_vertices)
        pool_np = np.ascontiguousarray(pool, dtype=np.int64)
        if not pool_np.flags.writeable:  # read-only pools (reference dataclasses) — torch needs a writable view
            pool_np = pool_np.copy()
        pool_dev = torch.from_numpy(pool_np).cuda()
        shuffled = gpu_stream.derive(ROLE_SHUFFLE).permutation_device(L, pool_dev).to(torch.int32)
        nb = math.ceil(L / B)
        H = len(self.cfg.fanouts)
        # the epoch's batch sizes and hop keys go to the device once: per window only
        # device-to-device copies, so no pageable copy stalls the host between windows
        counts = np.full(nb, B, dtype=np.int32)
        counts[-1] = L - (nb - 1) * B
        d_counts = torch.from_numpy(counts).cuda()
        d_keys = torch.from_numpy(batch_hop_keys(gpu_stream, 0, nb, H).view(np.int64)).cuda() if H else None
        sp = self.sampler
        W = sp.W
        for w0 in range(0, nb, W):
            w1 = min(nb, w0 + W)
            lo, hi = w0 * B, min(L, w1 * B)
            sp.active = w1 - w0
            sp.seeds.view(-1)[: hi - lo].copy_(shuffled[lo:hi])
            sp.counts[0, : w1 - w0].copy_(d_counts[w0:w1])
            if H:
                sp.keys[:, : w1 - w0].copy_(d_keys[w0:w1].t())
            sp.run(hot)
        return nb


def run_sampling_epoch(graph: CsrGraph, seed_pools, layout: CliqueLayout, cfg: SamplingConfig, seed: int,
                       epoch: int) -> list[GpuTrace]:
    """Replay one epoch of local-shuffle batching and sampling on every GPU of the
    layout (sampling.py:200-244); streams keyed by (seed, epoch, clique, gpu, batch, hop)."""
    n = graph.num_vertices
    root = KeyedRng(seed)
    traces = [
        GpuTrace(np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(n, np.int64)) for _ in range(layout.num_gpus)
    ]
    pools = [np.asarray(p, dtype=np.int64) for p in seed_pools]
    runner = None
    for ci, members in enumerate(layout.cliques):
        for li, gpu in enumerate(members):
            pool = pools[gpu]
            if len(pool) == 0:
                continue
            if runner is None:
                runner = EpochRunner(graph, cfg, max(len(p) for p in pools))
            hot = DeviceHotness(n)
            nb = runner.run(pool, root.derive(epoch, ci, li), hot)
            traces[gpu] = GpuTrace(
                hot.topo_reads.cpu().numpy(), hot.feat_lookups.cpu().numpy(), hot.edge_traversals.cpu().numpy(), nb
            )
    return traces


def run_presampling(graph: CsrGraph, tablets, layout: CliqueLayout, cfg: SamplingConfig,
                    spec: HardwareSpec) -> list[HotnessMatrices]:
    """presample_epochs epochs from the tablets -> per-clique hotness and N_TSUM
    (sampling.py:247-289). Counters accumulate in HBM across epochs; one copy out."""
    from .partition import TabletAssignment, assign_tablets

    pools = assign_tablets(tablets, layout) if isinstance(tablets, TabletAssignment) else list(tablets)
    if len(pools) != layout.num_gpus:
        raise ValueError("one seed pool per GPU required")
    for gpu, pool in enumerate(pools):
        if len(pool) == 0:
            warnings.warn(f"empty training tablet for gpu {gpu}; its hotness rows stay zero")
    pools = [np.asarray(p, dtype=np.int64) for p in pools]
    n = graph.num_vertices
    result = [
        HotnessMatrices(ci, np.zeros((len(m), n), np.int64), np.zeros((len(m), n), np.int64))
        for ci, m in enumerate(layout.cliques)
    ]
    if cfg.presample_epochs == 0 or all(len(p) == 0 for p in pools):
        return result
    runner = EpochRunner(graph, cfg, max(len(p) for p in pools))
    root = KeyedRng(cfg.seed)
    for ci, members in enumerate(layout.cliques):
        hot_rows = result[ci]
        for li, gpu in enumerate(members):
            if len(pools[gpu]) == 0:
                continue
            hot = DeviceHotness(n, spec)
            for epoch in range(cfg.presample_epochs):
                runner.run(pools[gpu], root.derive(epoch, ci, li), hot)
            hot_rows.topo_hotness[li] += hot.edge_traversals.cpu().numpy()
            hot_rows.feat_hotness[li] += hot.feat_lookups.cpu().numpy()
            hot_rows.sampling_txn_total += int(hot.txn_total.item())
    return result


def write_hotness(path, matrices: list[HotnessMatrices]) -> None:
    """u32 dump: per clique <I K_g><Q n>, H_T rows, H_F rows, <Q N_TSUM> (sampling.py:292-303)."""
    with open(path, "wb") as fh:
        for hot in matrices:
            if hot.topo_hotness.max(initial=0) > 0xFFFFFFFF or hot.feat_hotness.max(initial=0) > 0xFFFFFFFF:
                raise OverflowError("hotness counts exceed u32 dump format")
            fh.write(struct.pack("<IQ", hot.clique_size, hot.num_vertices))
            fh.write(hot.topo_hotness.astype("<u4").tobytes())
            fh.write(hot.feat_hotness.astype("<u4").tobytes())
            fh.write(struct.pack("<Q", hot.sampling_txn_total))


def read_hotness(path) -> list[HotnessMatrices]:
    """Inverse of write_hotness (sampling.py:306-326)."""
    data = open(path, "rb").read()
    out, pos = [], 0
    while pos < len(data):
        k, n = struct.unpack_from("<IQ", data, pos)
        pos += 12
        cells = k * n
        topo = np.frombuffer(data, "<u4", cells, pos).reshape(k, n).astype(np.int64)
        pos += 4 * cells
        feat = np.frombuffer(data, "<u4", cells, pos).reshape(k, n).astype(np.int64)
        pos += 4 * cells
        (txn,) = struct.unpack_from("<Q", data, pos)
        pos += 8
        out.append(HotnessMatrices(len(out), topo, feat, int(txn)))
    return out
