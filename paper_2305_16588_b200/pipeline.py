"""Per-GPU epoch pipeline: local shuffle -> windows of sampled, deduplicated,
relabelled and gathered mini-batches, all on the device.

This is Legion's batch generator + neighbour sampler + feature extractor for one
GPU over the reference's exact streams: the shuffle key is
root.derive(epoch, clique, gpu).derive(ROLE_SHUFFLE) and batch b's hop h key is
root.derive(epoch, clique, gpu).derive(ROLE_SAMPLE, b).derive(h)
(sampling.py:215-234). Host work per epoch is the key table (vectorised numpy)
and the launch sequence; no host round trip happens inside an epoch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cache import FeatureStore
from .graph import CsrGraph
from .rng import ROLE_SHUFFLE, KeyedRng
from .sampling import MAX_WINDOW, DeviceHotness, SamplingConfig, WindowSampler, batch_hop_keys, check_seed_pool

# kernels each stage launches (for the bench's gpu_launches count): the permutation is a
# histogram, a 3-kernel scan of the bucket counts, a scatter and the in-bucket rank/emit
LAUNCHES_PERMUTATION = 6


def _as_i64(key: int) -> int:
    """uint64 bit pattern -> the int64 a torch tensor stores."""
    key = int(key) & 0xFFFFFFFFFFFFFFFF
    return key - (1 << 64) if key >= 1 << 63 else key


def offsets_from_counts(counts, counts_ptr) -> tuple[torch.Tensor, np.ndarray]:
    """One hop's packed offsets from window_to_host's compact per-position counts:
    returns (offsets int32 [sum (F + 1)], offsets_ptr int64 [nb + 1]) laid out as the
    non-compact 'offsets'[h] / 'offsets_ptr'[h] (each batch's offsets start at 0)."""
    c = counts.numpy() if isinstance(counts, torch.Tensor) else np.asarray(counts)
    cp = np.asarray(counts_ptr, dtype=np.int64)
    nb = len(cp) - 1
    optr = cp + np.arange(nb + 1, dtype=np.int64)
    out = np.zeros(int(optr[-1]), dtype=np.int32)
    for b in range(nb):
        c0, c1 = int(cp[b]), int(cp[b + 1])
        out[optr[b] + 1 : optr[b + 1]] = np.cumsum(c[c0:c1], dtype=np.int64)
    return torch.from_numpy(out), optr


@dataclass
class EpochPlan:
    pool: torch.Tensor  # int64 [L] device
    shuffle_key: int
    keys: torch.Tensor  # int64 [nb, H] device (uint64 bit patterns)
    counts: torch.Tensor  # int32 [nb] device
    num_batches: int
    shuffle_key_dev: torch.Tensor | None = None  # int64 [1] device: the key read at run time (graphs)


class StageTimer:
    """CUDA events around each stage on the launching stream."""

    def __init__(self):
        self.events: dict[str, list] = {}

    def start(self, name: str):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        self.events.setdefault(name, []).append((e0, e1))
        return e1

    def summary(self) -> dict[str, tuple[int, float]]:
        """name -> (launch count, total ms); call after synchronising."""
        return {k: (len(v), sum(a.elapsed_time(b) for a, b in v)) for k, v in self.events.items()}

    def reset(self):
        self.events.clear()

    @staticmethod
    def hold(ms: float = 30.0, clock_ghz: float = 2.0) -> None:
        """Stall the current stream for ~ms (a device spin) so the host enqueues the
        whole epoch before the GPU starts it: stage events then bracket device time
        only, not host launch latency. Call right before a timed run_epoch."""
        torch.cuda._sleep(int(ms * 1e-3 * clock_ghz * 1e9))


class SampleGatherPipeline:
    """Sampling + dedup + relabel + three-tier gather for one GPU's seed pool.

    lanes > 1 is Legion's inter-batch pipeline: consecutive
    windows alternate between `lanes` independent sets of window buffers, each on its
    own CUDA stream, so one window's PCIe/HBM-bound gather overlaps the next
    window's ALU-bound sampling. Results are identical; only the schedule changes."""

    def __init__(self, graph: CsrGraph, cfg: SamplingConfig, store: FeatureStore | None, max_pool: int,
                 window: int | None = None, relabel: bool = True, feat_rows_cap: int | None = None,
                 placement: str = "hbm", topology=None, sparse_visited: bool | None = None, lanes: int = 1,
                 defer_host: bool | None = None, overlap_relabel: bool = True, mem_priority: bool = False):
        self.graph = graph
        self.cfg = cfg
        self.store = store
        B = cfg.batch_size
        nb = max(1, math.ceil(max_pool / B))
        self.window = min(nb, window or nb, MAX_WINDOW)
        if lanes < 1:
            raise ValueError("lanes must be >= 1")
        self.lane_samplers = []
        self.lane_features = []
        for _ in range(lanes):
            sp = WindowSampler(graph, cfg.fanouts, B, self.window, placement=placement, relabel=relabel,
                               unique_cap=feat_rows_cap, topology=topology, sparse_visited=sparse_visited)
            self.lane_samplers.append(sp)
            feats = None
            if store is not None:
                feats = torch.empty((self.window, sp.ucap, store.spec.dimension), dtype=torch.float32, device="cuda")
            self.lane_features.append(feats)
        self.lane_streams = [torch.cuda.Stream() for _ in range(lanes)] if lanes > 1 else []
        # defer_host: a window's host-tier rows are listed by the gather and read by a
        # second small-grid kernel in ascending address order (gc_gather_deferred,
        # GC_OPT_DEFER_ORDER). Random host rows are held to ~26 GB/s by the box's
        # host-side address translation; address order over a large window reads
        # faster. With lanes > 1 it runs on one high-priority stream; given a few fat
        # host-row CTAs (GC_OPT_DEFER_CTAS / GC_OPT_DEFER_ROWS, e.g. 32 x 256 rows) it
        # holds only those SMs and the other lane's sampling runs beside it: C3 64.3K ->
        # 112K batches/s with two lanes of 1536-batch windows
        # (profiles/r02_host_tier_pages.md). It pays with large windows, so it is off
        # unless asked for.
        self.defer_host = False if defer_host is None else bool(defer_host)
        self.host_stream = torch.cuda.Stream(priority=-1) if self.defer_host and lanes > 1 else None
        self.sampler = self.lane_samplers[0]
        self.features = self.lane_features[0]
        # relabel overlaps the gather on a side stream per lane (None: back to back), so
        # one lane's relabel never queues behind another lane's compaction
        # mem_priority: a window's memory-bound stages (dedup, relabel, gather) run on a
        # high-priority stream of its lane, so with lanes > 1 their CTAs take SM slots
        # ahead of the next window's ALU-bound hop expansion as those slots free up
        self.mem_streams = [torch.cuda.Stream(priority=-1) for _ in range(lanes)] if mem_priority else None
        prio = -1 if mem_priority else 0
        self._relabel_sides = [torch.cuda.Stream(priority=prio) for _ in range(lanes)] if overlap_relabel else None
        self._lane = 0
        self.feat_cap = self.sampler.ucap
        self.timer: StageTimer | None = None
        self.launches = 0
        self._graph = None  # run_epoch_graph: (CUDA graph, static plan, launches per replay)

    @property
    def lanes(self) -> int:
        return len(self.lane_samplers)

    # ------------------------------------------------------------------ host prep
    def plan_epoch(self, pool, gpu_stream: KeyedRng, validated: bool = False) -> EpochPlan:
        """validated=True: the caller has checked the ids already (e.g. once on the host
        for a pool it uploads every epoch), so a device pool is not read back here."""
        B = self.cfg.batch_size
        if not validated:
            check_seed_pool(pool, self.graph.num_vertices)
        pool_dev = pool if isinstance(pool, torch.Tensor) else torch.from_numpy(np.asarray(pool, np.int64)).cuda()
        L = pool_dev.numel()
        nb = math.ceil(L / B)
        keys = batch_hop_keys(gpu_stream, 0, nb, len(self.cfg.fanouts))
        counts = np.full(nb, B, dtype=np.int32)
        if nb:
            counts[-1] = L - (nb - 1) * B
        return EpochPlan(
            pool_dev,
            gpu_stream.derive(ROLE_SHUFFLE).key,
            torch.from_numpy(keys.view(np.int64)).cuda(),
            torch.from_numpy(counts).cuda(),
            nb,
        )

    # ------------------------------------------------------------------ device epoch
    def _stage(self, name):
        return self.timer.start(name) if self.timer is not None else None

    def run_epoch(self, plan: EpochPlan, on_window=None, hot: DeviceHotness | None = None) -> None:
        """Shuffle + all windows of one epoch; on_window(pipeline, first_batch, nbatches)
        is called after each window's device work has been enqueued (with lanes > 1,
        on that window's stream and with `sampler`/`features` pointing at its lane).
        On return the caller's stream is ordered after every window."""
        B, H = self.cfg.batch_size, len(self.cfg.fanouts)
        end = self._stage("shuffle")
        shuffled = KeyedRng(plan.shuffle_key).permutation_device(plan.pool.numel(), plan.pool,
                                                                 key_tensor=plan.shuffle_key_dev)
        self.launches += LAUNCHES_PERMUTATION
        if end is not None:
            end.record()
        main = torch.cuda.current_stream()
        if self.lane_streams:
            ready = torch.cuda.Event()
            ready.record(main)
            for st in self.lane_streams:
                st.wait_event(ready)
        for i, w0 in enumerate(range(0, plan.num_batches, self.window)):
            lane = i % self.lanes
            self._lane = lane
            self.sampler = self.lane_samplers[lane]
            self.features = self.lane_features[lane]
            if self.lane_streams:
                with torch.cuda.stream(self.lane_streams[lane]):
                    self._window(plan, shuffled, w0, on_window, hot)
            else:
                self._window(plan, shuffled, w0, on_window, hot)
        if self.lane_streams:
            for st in self.lane_streams:
                done = torch.cuda.Event()
                done.record(st)
                main.wait_event(done)
            # `shuffled` and the plan's tensors were used on the lane streams
            for st in self.lane_streams:
                shuffled.record_stream(st)

    def run_epoch_graph(self, plan: EpochPlan) -> None:
        """run_epoch as one CUDA-graph launch: the epoch's ~20 kernels (and the lanes'
        and relabel stream's fork/join) are captured on the first call and replayed
        after copying this epoch's inputs — pool, hop keys, batch sizes, shuffle key —
        into the captured static buffers. Same results as run_epoch; no host work or
        launch gaps between the kernels. The pool size must stay the same."""
        shape = (plan.pool.numel(), plan.num_batches)
        if self._graph is None or self._graph[1].pool.numel() != shape[0] \
                or self._graph[1].num_batches != shape[1]:
            static = EpochPlan(plan.pool.clone(), plan.shuffle_key, plan.keys.clone(), plan.counts.clone(),
                               plan.num_batches, torch.zeros(1, dtype=torch.int64, device="cuda"))
            static.shuffle_key_dev.fill_(_as_i64(plan.shuffle_key))
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):  # warm-up outside the capture (allocations, lazy init)
                self.run_epoch(static)
            torch.cuda.current_stream().wait_stream(side)
            before = self.launches
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.run_epoch(static)
            self._graph = (g, static, self.launches - before)
        g, static, per_replay = self._graph
        static.pool.copy_(plan.pool)
        static.keys.copy_(plan.keys)
        static.counts.copy_(plan.counts)
        static.shuffle_key_dev.fill_(_as_i64(plan.shuffle_key))
        g.replay()
        self.launches += per_replay

    def _window(self, plan: EpochPlan, shuffled: torch.Tensor, w0: int, on_window, hot) -> None:
        sp = self.sampler
        B, H = self.cfg.batch_size, len(self.cfg.fanouts)
        w1 = min(plan.num_batches, w0 + self.window)
        nb = w1 - w0
        lo, hi = w0 * B, min(plan.pool.numel(), w1 * B)
        sp.active = nb
        sp.seeds.view(-1)[: hi - lo].copy_(shuffled[lo:hi])
        sp.counts[0, :nb].copy_(plan.counts[w0:w1])
        if H:
            sp.keys[:, :nb].copy_(plan.keys[w0:w1].t())
        sp.expand(hot, timer=self.timer)
        self.launches += max(H, 1)
        if self.mem_streams is not None and self.timer is None:
            lane_stream = torch.cuda.current_stream()
            mem = self.mem_streams[self._lane]
            mem.wait_stream(lane_stream)
            with torch.cuda.stream(mem):
                self._memory_stages(sp, nb, hot, w0, on_window)
            lane_stream.wait_stream(mem)
            return
        self._memory_stages(sp, nb, hot, w0, on_window)

    def _memory_stages(self, sp, nb, hot, w0, on_window) -> None:
        H = len(self.cfg.fanouts)
        end = self._stage("unique_relabel")
        # relabel and gather both only need the compaction: with the side stream the two
        # HBM-bound passes share the GPU instead of running back to back
        side = self._relabel_sides[self._lane] if (self._relabel_sides and self.store is not None
                                                   and self.timer is None) else None
        sp.dedup(hot, relabel_stream=side)
        # compaction (1, 3 or 4 kernels, see gc_unique_compact_launches); one relabel per level
        self.launches += sp.lib.gc_unique_compact_launches(nb, sp.visited) + (H + 1 if sp.relabel else 0)
        if end is not None:
            end.record()
        if self.store is not None:
            end = self._stage("gather")
            self.store.gather(sp.unique, sp.ucount, self.features, num_batches=nb, deferred=self.defer_host,
                              host_stream=self.host_stream)
            self.launches += 1
            if end is not None:
                end.record()
        if side is not None:
            joined = torch.cuda.Event()
            joined.record(side)
            torch.cuda.current_stream().wait_event(joined)
        if on_window is not None:
            on_window(self, w0, nb)

    def check_capacity(self, reset: bool = False) -> int:
        """Raise OverflowError if any batch since the last reset had more distinct
        vertices than feat_rows_cap (its rows would have been truncated); one sync."""
        return max(sp.check_capacity(reset) for sp in self.lane_samplers)

    # ------------------------------------------------------------------ host delivery
    def window_to_host(self, nb: int, staging: dict | None = None, compact_ids: bool = False,
                       wait: bool = True) -> dict:
        """The last window's results in pinned host memory, packed batch after batch.

        The device buffers are padded [batch, capacity]; each array's per-batch
        segments are first packed on the device (a masked gather, HBM-speed), so the
        PCIe link carries one large copy per array instead of 2 + 2H small copies per
        batch. Returns host tensors (views into `staging`, valid until the next call):
        'unique' int32 [sum U], 'features' f32 [sum U, D] (with a feature store),
        'offsets'[h] int32 [sum (F_h + 1)], 'local'[h] int32 [sum T_h] (global
        neighbour ids when the pipeline does not relabel), and the batch boundaries
        'unique_ptr', 'offsets_ptr'[h], 'local_ptr'[h] (int64 numpy [nb + 1]).
        compact_ids: relabelled ids of a window whose batches all have <= 65536
        distinct vertices travel as 16-bit values ('local'[h] int16 holding the uint16
        bit pattern, out['local_bits'] = 16), and, when every fanout is <= 255, each
        hop's offsets travel as per-position u8 sample counts ('counts'[h] uint8
        [sum F_h] with 'counts_ptr'[h]; offsets_from_counts() rebuilds 'offsets'[h]) —
        less than half the PCIe bytes of u32 ids and offsets at C2.
        The packing is sync-free (segment rows from the host-side sizes) and each
        array's D2H copy runs on a copy stream while the next array is packed; the
        kernels enqueued after this call may overwrite the window's buffers at once
        (the copies read the packed arrays). Reads the sizes once (a sync). wait=False:
        returns before the copies land — out['ready'] (a CUDA event on the copy
        stream) must be synchronised before the host arrays are read or the staging
        buffers reused, which lets the next window's sampling overlap the D2H."""
        sp = self.sampler
        st = {} if staging is None else staging
        main = torch.cuda.current_stream()
        # the window's sizes, read through mapped memory by SM stores: a DMA read would
        # queue behind the previous window's bulk copies still in the copy engine
        sizes = torch.cat([sp.counts[:, :nb].reshape(-1), sp.ucount[:nb]])
        hs = st.get("_sizes")
        if hs is None or hs.numel() < sizes.numel():
            hs = st["_sizes"] = torch.empty(max(sizes.numel(), 1024), dtype=torch.int32, pin_memory=True)
        _lib.check(_lib.lib().gc_copy_d2h_mapped(sizes.data_ptr(), hs.data_ptr(), sizes.numel() * 4,
                                                 _lib.stream_handle(main)), "copy_d2h_mapped")
        done = torch.cuda.Event()
        done.record(main)
        done.synchronize()
        flat = hs[: sizes.numel()].numpy().astype(np.int64)
        counts = flat[: (sp.H + 1) * nb].reshape(sp.H + 1, nb)
        ucount = flat[(sp.H + 1) * nb :]
        if nb and int(ucount.max()) > sp.ucap:
            raise OverflowError(f"a batch has {int(ucount.max())} distinct vertices but the unique/gather "
                                f"capacity is {sp.ucap}: raise feat_rows_cap")
        copy = st.get("_copy_stream")
        if copy is None:
            copy = st["_copy_stream"] = torch.cuda.Stream()
        u16 = compact_ids and sp.local_nbrs is not None and (not nb or int(ucount.max()) <= 1 << 16)

        def ptr(sizes):
            return np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)

        lib = _lib.lib()

        def dev_buffer(key, shape, dtype):
            # persistent per staging set (the caller alternates sets and waits for a set's
            # copies before reusing it): no allocator traffic inside an epoch
            t = st.get(key)
            if t is None or t.shape[0] < shape[0] or t.shape[1:] != shape[1:] or t.dtype != dtype:
                rows = max(shape[0] + shape[0] // 4, 1)
                t = torch.empty((rows,) + tuple(shape[1:]), dtype=dtype, device="cuda")
                st[key] = t
            return t

        def pack(name, buf, sizes, narrow=False, counts=False):
            # one gc_pack_segments launch: batch b's first sizes[b] rows of the padded
            # [nb, cap, ...] buffer land at row ptr[b] of a packed device array; ids
            # stored as u16 (int16) travel as such when narrow, else widen to int32;
            # counts: offsets become the u8 differences of consecutive entries
            total = int(sizes.sum())
            u16_in = buf.dtype == torch.int16
            if counts:
                dtype, mode = torch.uint8, 4
            else:
                dtype = torch.int16 if narrow else (torch.int32 if u16_in else buf.dtype)
                mode = (2 if narrow else 3) if u16_in else (1 if narrow else 0)
            tail = tuple(buf.shape[2:])
            packed = dev_buffer(f"_dev_{name}", (total,) + tail, dtype)[:total]
            if total:
                p = ptr(sizes)
                hp = st.get(f"_ptr_{name}")
                if hp is None or hp.numel() < p.size:
                    hp = st[f"_ptr_{name}"] = torch.empty(max(p.size, 1024), dtype=torch.int64, pin_memory=True)
                hp[: p.size].copy_(torch.from_numpy(p))
                dp = dev_buffer(f"_dptr_{name}", (hp.numel(),), torch.int64)
                dp[: p.size].copy_(hp[: p.size], non_blocking=True)
                row_bytes = buf.element_size() * int(np.prod(tail, dtype=np.int64))
                _lib.check(lib.gc_pack_segments(buf.data_ptr(), buf.stride(0) * buf.element_size(), row_bytes,
                                                dp.data_ptr(), nb, int(sizes.max()), mode, packed.data_ptr(),
                                                _lib.stream_handle(main)), "pack_segments")
            host = st.get(name)
            if host is None or host.shape[0] < total or host.shape[1:] != packed.shape[1:] or host.dtype != packed.dtype:
                # 25% slack: pinned allocations are slow, so a slightly larger window later reuses it
                rows = max(total + total // 4, 1)
                host = torch.empty((rows,) + tuple(packed.shape[1:]), dtype=packed.dtype, pin_memory=True)
                st[name] = host
            # the copy stream moves this array over PCIe while the next one is packed
            ev = torch.cuda.Event()
            ev.record(main)
            copy.wait_event(ev)
            with torch.cuda.stream(copy):
                host[:total].copy_(packed, non_blocking=True)
            return host[:total]

        as_counts = compact_ids and max(sp.fanouts, default=0) <= 255
        out = {"unique_ptr": ptr(ucount), "offsets_ptr": [], "local_ptr": [], "local": [],
               "local_bits": 16 if u16 else 32}
        out.update({"counts": [], "counts_ptr": []} if as_counts else {"offsets": []})
        out["unique"] = pack("unique", sp.unique, ucount)
        if self.store is not None:
            out["features"] = pack("features", self.features, ucount)
        for h in range(sp.H):
            f, t = counts[h] + 1, counts[h + 1]
            out["offsets_ptr"].append(ptr(f))
            out["local_ptr"].append(ptr(t))
            if as_counts:
                out["counts_ptr"].append(ptr(counts[h]))
                out["counts"].append(pack(f"counts{h}", sp.offsets[h], counts[h], counts=True))
            else:
                out["offsets"].append(pack(f"offsets{h}", sp.offsets[h], f))
            ids = sp.local_nbrs[h] if sp.local_nbrs is not None else sp.nbrs[h]  # relabel=False: global ids
            out["local"].append(pack(f"local{h}", ids, t, narrow=u16))
        ready = torch.cuda.Event()
        ready.record(copy)
        out["ready"] = ready
        if wait:
            ready.synchronize()
        return out

    # ------------------------------------------------------------------ accounting
    def window_bytes(self, nb: int) -> dict[str, int]:
        """Algorithmic bytes of the last window by kernel stage; syncs.

        hop h: frontier ids 4F + row-offset pair 16F + selected columns 4T read,
               neighbours 4T + offsets 4(F+1) written
        unique+relabel: distinct ids 4U written; every sampled id read 4 B and its
               local index written 4 B
        gather: U rows read from their tier and U rows written"""
        sp = self.sampler
        counts = sp.counts[:, :nb].cpu().numpy().astype(np.int64)  # [H+1, nb]
        ucount = sp.ucount[:nb].cpu().numpy().astype(np.int64)
        F = counts[:-1].sum(axis=1)  # per hop frontier positions
        T = counts[1:].sum(axis=1)  # per hop sampled neighbours
        hop = 4 * F + 16 * F + 4 * T + 4 * T + 4 * (F + nb)
        ids = int(counts.sum())
        dedup = 4 * int(ucount.sum()) + (8 * ids if sp.relabel else 0)
        row = self.store.spec.row_bytes if self.store is not None else 0
        gather = 2 * row * int(ucount.sum())
        out = {"sampling": int(hop.sum()), "dedup": dedup, "gather": gather, "unique_rows": int(ucount.sum()),
               "sampled": int(T.sum())}
        for h in range(len(hop)):
            out[f"hop_expand.h{h}"] = int(hop[h])
        return out
