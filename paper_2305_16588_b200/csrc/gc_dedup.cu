// K3 unique + relabel: BatchSample.distinct_vertices (sampling.py:73-75) is np.unique,
// i.e. the sorted distinct ids. Every emitted vertex marks a per-batch visited bitmap
// inside hop_expand, so the sorted unique list falls out of one ordered popcount scan
// of the bitmap (no sort). The per-word exclusive popcount, stored interleaved with
// the word itself as a rank table {prefix, bits}, is the relabel map:
// local(u) = prefix[u >> 5] + popc(bits[u >> 5] & lanes-below(u)) — one 8-byte load.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "gc_common.cuh"

namespace gc {

constexpr int kUniqThreads = 256;
constexpr int kWordsPerThread = 4;
constexpr int kWordsPerTile = kUniqThreads * kWordsPerThread;

struct UniqueParams {
    uint32_t* bm;
    uint64_t bwords;
    uint32_t tiles_per_batch;
    uint32_t* uniq;
    uint64_t ustride;
    uint32_t* ucount;
    uint2* rank;
    uint64_t* feat;
    int clear;
    uint32_t* tile_count;  // [W][tiles] distinct ids per tile, then their exclusive prefix
};

// Dense compaction in three passes over tiles of 1024 words (no inter-tile wait; a
// single pass with a decoupled look-back spent 69% of its time at barriers behind
// the look-back convoy): tile popcounts, a per-batch scan of them, then the ordered
// emission of every tile from its known offset.
__global__ void __launch_bounds__(kUniqThreads) k_unique_counts(UniqueParams p) {
    using Reduce = cub::BlockReduce<uint32_t, kUniqThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    const uint32_t b = blockIdx.y, t = blockIdx.x;
    const uint64_t w0 = (uint64_t)t * kWordsPerTile + (uint64_t)threadIdx.x * kWordsPerThread;
    uint4 x = make_uint4(0, 0, 0, 0);
    if (w0 < p.bwords) x = *reinterpret_cast<const uint4*>(p.bm + b * p.bwords + w0);  // bwords % 4 == 0
    const uint32_t c = Reduce(tmp).Sum(__popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w));
    if (threadIdx.x == 0) p.tile_count[(uint64_t)b * p.tiles_per_batch + t] = c;
}

__global__ void __launch_bounds__(1024) k_unique_tile_scan(UniqueParams p) {
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t s_run;
    const uint32_t b = blockIdx.x;
    uint32_t* cnt = p.tile_count + (uint64_t)b * p.tiles_per_batch;
    if (threadIdx.x == 0) s_run = 0;
    __syncthreads();
    for (uint32_t base = 0; base < p.tiles_per_batch; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < p.tiles_per_batch ? cnt[i] : 0u;
        uint32_t excl, total;
        Scan(tmp).ExclusiveSum(v, excl, total);
        if (i < p.tiles_per_batch) cnt[i] = s_run + excl;
        __syncthreads();
        if (threadIdx.x == 0) s_run += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) p.ucount[b] = s_run;
}

__global__ void __launch_bounds__(kUniqThreads) k_unique(UniqueParams p) {
    using Scan = cub::BlockScan<uint32_t, kUniqThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    const uint32_t b = blockIdx.y, t = blockIdx.x;
    const int tid = threadIdx.x;
    const uint64_t w0 = (uint64_t)t * kWordsPerTile + (uint64_t)tid * kWordsPerThread;
    uint32_t* row = p.bm + b * p.bwords;
    const uint32_t tile_base = p.tile_count[(uint64_t)b * p.tiles_per_batch + t];
    uint4 x = make_uint4(0, 0, 0, 0);
    if (w0 < p.bwords) x = *reinterpret_cast<const uint4*>(row + w0);
    const uint32_t c0 = __popc(x.x), c1 = __popc(x.y), c2 = __popc(x.z), c3 = __popc(x.w);
    uint32_t excl, total;
    Scan(scan_tmp).ExclusiveSum(c0 + c1 + c2 + c3, excl, total);
    if (total == 0) return;
    const uint32_t base = tile_base + excl;
    if (w0 < p.bwords) {
        // relabel only looks up words holding a present id: empty words need no entry
        if (p.rank && (x.x | x.y | x.z | x.w)) {
            uint4* rt = reinterpret_cast<uint4*>(p.rank + b * p.bwords + w0);
            if (x.x | x.y) rt[0] = make_uint4(base, x.x, base + c0, x.y);
            if (x.z | x.w) rt[1] = make_uint4(base + c0 + c1, x.z, base + c0 + c1 + c2, x.w);
        }
        uint32_t* out = p.uniq + b * p.ustride;
        uint32_t pos = base;
        const uint32_t words[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t w = words[k];
            const uint32_t vbase = (uint32_t)((w0 + k) * 32);
            while (w) {
                const uint32_t u = vbase + (__ffs(w) - 1);
                // capacity guard: ucount still reports the true count, so the caller
                // sees ucount > unique_stride and raises (rows past the cap are dropped)
                if (pos < p.ustride) out[pos] = u;
                ++pos;
                if (p.feat) atomicAdd((unsigned long long*)(p.feat + u), 1ull);
                w &= w - 1;
            }
        }
        if (p.clear && (x.x | x.y | x.z | x.w)) *reinterpret_cast<uint4*>(row + w0) = make_uint4(0, 0, 0, 0);
    }
}

// Dense compaction with one 1024-thread CTA per batch, for windows of at least a
// GPU's worth of batches (C2: 235): the CTA walks its batch's bitmap in 4096-word
// chunks (the next chunk's loads in flight while the current one is scanned and
// emitted), so there is one launch instead of three and no per-tile CTA turnover.
// Same outputs as k_unique_counts + k_unique_tile_scan + k_unique.
constexpr int kFusedThreads = 1024;
constexpr uint32_t kFusedWords = kFusedThreads * kWordsPerThread;

__global__ void __launch_bounds__(kFusedThreads) k_unique_batch(UniqueParams p) {
    __shared__ uint32_t s_warp[2][32];
    const uint32_t b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t* row = p.bm + b * p.bwords;
    uint32_t* out = p.uniq + b * p.ustride;
    uint4* rt = p.rank ? reinterpret_cast<uint4*>(p.rank + b * p.bwords) : nullptr;
    uint32_t run = 0;
    uint64_t w0 = (uint64_t)tid * kWordsPerThread;
    uint4 x = w0 < p.bwords ? *reinterpret_cast<const uint4*>(row + w0) : make_uint4(0, 0, 0, 0);
    for (uint32_t it = 0; (uint64_t)it * kFusedWords < p.bwords; ++it) {
        const uint64_t wn = w0 + kFusedWords;
        const uint4 xn = wn < p.bwords ? *reinterpret_cast<const uint4*>(row + wn) : make_uint4(0, 0, 0, 0);
        const uint32_t c0 = __popc(x.x), c1 = __popc(x.y), c2 = __popc(x.z), c3 = __popc(x.w);
        const uint32_t cnt = c0 + c1 + c2 + c3;
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t* sw = s_warp[it & 1];  // alternating: no barrier before the next chunk's writes
        if (lane == 31) sw[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            uint32_t v = sw[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, v, o);
                if (lane >= o) v += y;
            }
            sw[lane] = v;
        }
        __syncthreads();
        const uint32_t base = run + (wid ? sw[wid - 1] : 0u) + incl - cnt;
        run += sw[31];
        if (cnt) {
            if (rt) {
                if (x.x | x.y) rt[w0 / 2] = make_uint4(base, x.x, base + c0, x.y);
                if (x.z | x.w) rt[w0 / 2 + 1] = make_uint4(base + c0 + c1, x.z, base + c0 + c1 + c2, x.w);
            }
            uint32_t pos = base;
            const uint32_t words[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t w = words[k];
                const uint32_t vbase = (uint32_t)((w0 + k) * 32);
                while (w) {
                    const uint32_t u = vbase + (__ffs(w) - 1);
                    if (pos < p.ustride) out[pos] = u;  // capacity guard, as in k_unique
                    ++pos;
                    if (p.feat) atomicAdd((unsigned long long*)(p.feat + u), 1ull);
                    w &= w - 1;
                }
            }
            if (p.clear) *reinterpret_cast<uint4*>(row + w0) = make_uint4(0, 0, 0, 0);
        }
        x = xn;
        w0 = wn;
    }
    if (tid == 0) p.ucount[b] = run;
}

// Sparse compaction, fully parallel over the non-empty 32-word blocks (1024 vertices):
//   k_block_lists   one CTA per batch: summary bits -> ascending list of non-empty
//                   blocks (and the summary is cleared as it is read)
//   k_block_counts  warp per listed block: one coalesced 128-byte load, popcount
//   k_block_scan    one CTA per batch: exclusive scan of its block counts (the
//                   output offset of every block; ucount)
//   k_block_emit    warp per listed block: ids in ascending order, rank-table entries,
//                   the words it consumed cleared.
// Work is O(distinct blocks + n/32768) per batch instead of O(n/32), with no barrier or
// inter-block wait in the per-block passes. (A single pass with a decoupled look-back
// across chunks of blocks was measured at 32 ms per C3 epoch: with one wave of
// persistent CTAs every chunk's look-back walks back through the whole wave; a
// chunk-granular two-pass version at 16 ms.)
constexpr int kBlockWarps = kUniqThreads / 32;
#ifndef GC_BLOCKS_IN_FLIGHT
#define GC_BLOCKS_IN_FLIGHT 8  // C3 dedup+relabel 15.1 -> 13.6 ms per epoch (16: 14.7)
#endif
// listed blocks per warp per step (independent load chains): C3's touched blocks hold
// ~1 id each, so the passes are latency-bound and want many chains per warp
constexpr int kBlocksInFlight = GC_BLOCKS_IN_FLIGHT;

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t& total) {
    const int lane = threadIdx.x & 31;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(kFull, x, 31);
    return x - v;
}

struct SparseParams {
    uint32_t* bm;
    uint64_t bwords;
    uint32_t* sm;
    uint64_t swords;
    uint32_t num_batches;
    uint32_t* lists;     // [W][list_stride] non-empty block ids
    uint64_t list_stride;
    uint32_t* nblocks;   // [W]
    uint32_t* bcount;    // [W][list_stride] distinct ids per listed block, then their exclusive prefix
    uint32_t* uniq;
    uint64_t ustride;
    uint32_t* ucount;
    uint2* rank;
    uint64_t* feat;
    int clear;
};

__global__ void __launch_bounds__(kUniqThreads) k_block_lists(SparseParams p) {
    using Scan = cub::BlockScan<uint32_t, kUniqThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t s_run;
    const uint32_t b = blockIdx.x;
    uint32_t* srow = p.sm + b * p.swords;
    uint32_t* list = p.lists + b * p.list_stride;
    if (threadIdx.x == 0) s_run = 0;
    __syncthreads();
    for (uint64_t base = 0; base < p.swords; base += kUniqThreads) {
        const uint64_t sw = base + threadIdx.x;
        const uint32_t s = sw < p.swords ? srow[sw] : 0u;
        uint32_t excl, total;
        Scan(tmp).ExclusiveSum((uint32_t)__popc(s), excl, total);
        uint32_t pos = s_run + excl;
        for (uint32_t m = s; m; m &= m - 1u) list[pos++] = (uint32_t)(sw * 32 + (__ffs(m) - 1));
        if (p.clear && s) srow[sw] = 0u;
        __syncthreads();
        if (threadIdx.x == 0) s_run += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) p.nblocks[b] = s_run;
}

// grid (x, W): the warps of batch b's CTAs stride over its listed blocks,
// kBlocksInFlight at a time
__global__ void __launch_bounds__(kUniqThreads) k_block_counts(SparseParams p) {
    const uint32_t b = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const uint32_t nb = p.nblocks[b];
    const uint32_t* list = p.lists + b * p.list_stride;
    const uint32_t* row = p.bm + b * p.bwords;
    uint32_t* cnt = p.bcount + b * p.list_stride;
    const uint32_t warps = gridDim.x * kBlockWarps;
    for (uint32_t i0 = (blockIdx.x * kBlockWarps + (threadIdx.x >> 5)) * kBlocksInFlight; i0 < nb;
         i0 += warps * kBlocksInFlight) {
        uint32_t x[kBlocksInFlight];
#pragma unroll
        for (int k = 0; k < kBlocksInFlight; ++k) {
            x[k] = 0u;
            if (i0 + k < nb) {
                const uint64_t wi = (uint64_t)list[i0 + k] * 32 + lane;
                if (wi < p.bwords) x[k] = row[wi];
            }
        }
#pragma unroll
        for (int k = 0; k < kBlocksInFlight; ++k) {
            const uint32_t c = __reduce_add_sync(kFull, (uint32_t)__popc(x[k]));
            if (lane == 0 && i0 + k < nb) cnt[i0 + k] = c;
        }
    }
}

__global__ void __launch_bounds__(1024) k_block_scan(SparseParams p) {
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t s_run;
    const uint32_t b = blockIdx.x;
    const uint32_t nb = p.nblocks[b];
    uint32_t* cnt = p.bcount + b * p.list_stride;
    if (threadIdx.x == 0) s_run = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nb; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < nb ? cnt[i] : 0u;
        uint32_t excl, total;
        Scan(tmp).ExclusiveSum(v, excl, total);
        if (i < nb) cnt[i] = s_run + excl;  // in place: count -> exclusive prefix
        __syncthreads();
        if (threadIdx.x == 0) s_run += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) p.ucount[b] = s_run;
}

__global__ void __launch_bounds__(kUniqThreads) k_block_emit(SparseParams p) {
    const uint32_t b = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const uint32_t nb = p.nblocks[b];
    const uint32_t* list = p.lists + b * p.list_stride;
    uint32_t* row = p.bm + b * p.bwords;
    const uint32_t* pre = p.bcount + b * p.list_stride;
    uint32_t* out = p.uniq + b * p.ustride;
    uint2* rt = p.rank ? p.rank + b * p.bwords : nullptr;
    const uint32_t warps = gridDim.x * kBlockWarps;
    for (uint32_t i0 = (blockIdx.x * kBlockWarps + (threadIdx.x >> 5)) * kBlocksInFlight; i0 < nb;
         i0 += warps * kBlocksInFlight) {
        uint32_t x[kBlocksInFlight], base[kBlocksInFlight], blk[kBlocksInFlight];
#pragma unroll
        for (int k = 0; k < kBlocksInFlight; ++k) {
            x[k] = 0u;
            blk[k] = 0;
            base[k] = 0;
            if (i0 + k < nb) {
                blk[k] = list[i0 + k];
                base[k] = pre[i0 + k];
                const uint64_t w = (uint64_t)blk[k] * 32 + lane;
                if (w < p.bwords) x[k] = row[w];
            }
        }
#pragma unroll
        for (int k = 0; k < kBlocksInFlight; ++k) {
            uint32_t tot;
            uint32_t pos = base[k] + warp_excl_scan((uint32_t)__popc(x[k]), tot);
            if (x[k]) {
                const uint64_t wik = (uint64_t)blk[k] * 32 + lane;
                if (rt) rt[wik] = make_uint2(pos, x[k]);
                const uint32_t vbase = (uint32_t)(wik * 32);
                for (uint32_t w = x[k]; w; w &= w - 1u) {
                    const uint32_t u = vbase + (__ffs(w) - 1);
                    if (pos < p.ustride) out[pos] = u;  // capacity guard (see k_unique)
                    ++pos;
                    if (p.feat) atomicAdd((unsigned long long*)(p.feat + u), 1ull);
                }
                if (p.clear) row[wik] = 0u;
            }
        }
    }
}

struct SparseLayout {
    size_t lists, nblocks, bcount, total;
    uint64_t list_stride;
};

static SparseLayout sparse_layout(uint32_t W, const gc_visited_t* v) {
    SparseLayout L{};
    L.list_stride = v->summary_words * 32;
    size_t off = 0;
    L.lists = off; off = align_up(off + (size_t)W * L.list_stride * 4, 256);
    L.nblocks = off; off = align_up(off + (size_t)W * 4, 256);
    L.bcount = off; off = align_up(off + (size_t)W * L.list_stride * 4, 256);
    L.total = off;
    return L;
}

__device__ __forceinline__ uint32_t rank_of(const uint2* __restrict__ rt, uint32_t u) {
    const uint2 e = __ldg(rt + (u >> 5));
    return e.x + __popc(e.y & ((1u << (u & 31)) - 1u));
}

#ifndef GC_RELABEL_GROUPS
#define GC_RELABEL_GROUPS 3  // C2 unique+relabel 0.461 -> 0.449 ms (2: 0.478 in this form, 4: 0.454)
#endif
constexpr int kRelabelGroups = GC_RELABEL_GROUPS;

// VEC ids per thread per step (16-byte streaming loads when the batch stride keeps
// rows 16-byte aligned), so VEC independent rank-table loads are in flight. Local ids
// are stored as OUT (u32, or u16 when every batch of the window has at most 65536
// distinct vertices: a quarter less traffic for the pass, which moves 4 + sizeof(OUT)
// bytes per sampled id).
template <int VEC, typename OUT>
__global__ void k_relabel(const uint32_t* __restrict__ ids, uint64_t stride, const uint32_t* __restrict__ count,
                          const uint2* __restrict__ rank, uint64_t bwords, OUT* __restrict__ local) {
    const uint32_t b = blockIdx.y;
    const uint32_t c = count[b];
    const uint2* rt = rank + b * bwords;
    const uint32_t* in = ids + b * stride;
    OUT* out = local + b * stride;
    if constexpr (VEC == 4) {
        const uint32_t c4 = c / 4;
        const uint32_t step = gridDim.x * blockDim.x;
        // kRelabelGroups 16-byte groups per thread per step: 4 * kRelabelGroups
        // independent rank-table loads in flight
        for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < c4; k += kRelabelGroups * step) {
            uint4 u[kRelabelGroups];
#pragma unroll
            for (int j = 0; j < kRelabelGroups; ++j)
                u[j] = k + j * step < c4 ? __ldcs(reinterpret_cast<const uint4*>(in) + k + j * step)
                                         : make_uint4(0, 0, 0, 0);
            uint4 r[kRelabelGroups];
#pragma unroll
            for (int j = 0; j < kRelabelGroups; ++j) {  // all rank loads before any store
                r[j].x = rank_of(rt, u[j].x);
                r[j].y = rank_of(rt, u[j].y);
                r[j].z = rank_of(rt, u[j].z);
                r[j].w = rank_of(rt, u[j].w);
            }
#pragma unroll
            for (int j = 0; j < kRelabelGroups; ++j) {
                if (k + j * step >= c4) continue;
                if constexpr (sizeof(OUT) == 4) {
                    __stcs(reinterpret_cast<uint4*>(out) + k + j * step, r[j]);
                } else {  // four u16 in one 8-byte store
                    const uint2 v = make_uint2((r[j].x & 0xFFFFu) | (r[j].y << 16), (r[j].z & 0xFFFFu) | (r[j].w << 16));
                    __stcs(reinterpret_cast<uint2*>(out) + k + j * step, v);
                }
            }
        }
        const uint32_t k = c4 * 4 + blockIdx.x * blockDim.x + threadIdx.x;
        if (k < c) out[k] = (OUT)rank_of(rt, in[k]);
    } else {
        for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < c; k += gridDim.x * blockDim.x)
            out[k] = (OUT)rank_of(rt, __ldcs(in + k));
    }
}

__global__ void k_bitmap_clear(uint32_t* bm, uint64_t bwords, uint32_t* sm, uint64_t swords,
                               const uint32_t* __restrict__ uniq, uint64_t ustride, const uint32_t* __restrict__ ucount) {
    const uint32_t b = blockIdx.y;
    // only the first unique_stride ids were written (capacity guard of the compaction)
    const uint32_t c = (uint64_t)ucount[b] < ustride ? ucount[b] : (uint32_t)ustride;
    uint32_t* row = bm + b * bwords;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < c; k += gridDim.x * blockDim.x) {
        const uint32_t u = uniq[b * ustride + k];
        row[u >> 5] = 0u;
        if (sm) sm[b * swords + (u >> 15)] = 0u;
    }
}

__global__ void k_mark(const uint32_t* __restrict__ ids, uint64_t stride, const uint32_t* __restrict__ count,
                       uint32_t* bm, uint64_t bwords, uint32_t* sm, uint64_t swords) {
    const uint32_t b = blockIdx.y;
    const uint32_t c = count[b];
    uint32_t* row = bm + b * bwords;
    uint32_t* srow = sm ? sm + b * swords : nullptr;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < c; k += gridDim.x * blockDim.x)
        mark_visited(row, srow, ids[b * stride + k]);
}

// GC_OPT_UNIQUE_BATCH_CTAS: windows of at least this many batches take the
// CTA-per-batch dense compaction (0: the SM count)
static int g_unique_batch_min = 0;
void set_unique_batch_min(int v) { g_unique_batch_min = v; }

static unsigned uniq_tiles(const gc_visited_t* v) {
    uint64_t t = (v->words + kWordsPerTile - 1) / kWordsPerTile;
    return t ? (unsigned)t : 1u;
}

static unsigned grid_x(uint32_t max_count, int block) {
    uint64_t g = ((uint64_t)max_count + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 1024) g = 1024;
    return (unsigned)g;
}

}  // namespace gc

namespace gc {
template <typename OUT>
static int relabel(const uint32_t* d_ids, uint64_t ids_stride, const uint32_t* d_ids_count, uint32_t max_count,
                   uint32_t num_batches, const uint32_t* d_rank_table, uint64_t bitmap_words, OUT* d_local,
                   void* stream, const char* what) {
    GC_REQUIRE(num_batches < 65536, GC_ERR_VALUE, "gc_relabel: at most 65535 batches per call");
    if (num_batches == 0 || max_count == 0) return GC_OK;
    const auto* rt = reinterpret_cast<const uint2*>(d_rank_table);
    const bool vec = ids_stride % 4 == 0 && (uintptr_t)d_ids % 16 == 0 && (uintptr_t)d_local % (4 * sizeof(OUT)) == 0;
    if (vec) {
        dim3 grid(grid_x((max_count + 4 * kRelabelGroups - 1) / (4 * kRelabelGroups), 256), num_batches);
        k_relabel<4, OUT><<<grid, 256, 0, as_stream(stream)>>>(d_ids, ids_stride, d_ids_count, rt, bitmap_words,
                                                               d_local);
    } else {
        dim3 grid(grid_x(max_count, 256), num_batches);
        k_relabel<1, OUT><<<grid, 256, 0, as_stream(stream)>>>(d_ids, ids_stride, d_ids_count, rt, bitmap_words,
                                                               d_local);
    }
    GC_CHECK_LAUNCH(what);
    return GC_OK;
}

}  // namespace gc

using namespace gc;

extern "C" {

uint64_t gc_bitmap_words(int64_t num_vertices) {
    uint64_t w = ((uint64_t)(num_vertices > 0 ? num_vertices : 0) + 31) / 32;
    return (w + 3) / 4 * 4;
}

uint64_t gc_summary_words(int64_t num_vertices) {
    const uint64_t blocks = (gc_bitmap_words(num_vertices) + 31) / 32;
    return ((blocks + 31) / 32 + 3) / 4 * 4;
}

size_t gc_unique_temp_bytes(uint32_t num_batches, const gc_visited_t* visited) {
    if (!visited) return 0;
    if (visited->summary) return sparse_layout(num_batches, visited).total;
    return align_up((size_t)num_batches * uniq_tiles(visited) * sizeof(uint32_t), 256);
}

int gc_unique_compact(const gc_visited_t* visited, uint32_t num_batches, uint32_t* d_unique,
                      uint64_t unique_stride, uint32_t* d_unique_count, uint32_t* d_rank_table,
                      uint64_t* d_feat_lookups, int clear_bitmap, void* d_temp, size_t temp_bytes,
                      void* stream) {
    GC_REQUIRE(visited && visited->bitmap, GC_ERR_VALUE, "gc_unique_compact: visited set is null");
    GC_REQUIRE(visited->words % 4 == 0, GC_ERR_VALUE, "gc_unique_compact: bitmap words must be a multiple of 4");
    GC_REQUIRE(!visited->summary || visited->summary_words * 32 * 32 >= visited->words, GC_ERR_VALUE,
               "gc_unique_compact: summary too small for the bitmap");
    if (num_batches == 0) return GC_OK;
    const size_t need = gc_unique_temp_bytes(num_batches, visited);
    GC_REQUIRE(d_temp && temp_bytes >= need, GC_ERR_VALUE, "gc_unique_compact: temp buffer too small");
    cudaStream_t s = as_stream(stream);
    if (visited->summary) {
        const SparseLayout L = sparse_layout(num_batches, visited);
        char* t = static_cast<char*>(d_temp);
        SparseParams q{};
        q.bm = visited->bitmap;
        q.bwords = visited->words;
        q.sm = visited->summary;
        q.swords = visited->summary_words;
        q.num_batches = num_batches;
        q.lists = reinterpret_cast<uint32_t*>(t + L.lists);
        q.list_stride = L.list_stride;
        q.nblocks = reinterpret_cast<uint32_t*>(t + L.nblocks);
        q.bcount = reinterpret_cast<uint32_t*>(t + L.bcount);
        q.uniq = d_unique;
        q.ustride = unique_stride;
        q.ucount = d_unique_count;
        q.rank = reinterpret_cast<uint2*>(d_rank_table);
        q.feat = d_feat_lookups;
        q.clear = clear_bitmap;
        // the block lists need the summary; it is cleared as it is read only when the
        // bitmap is cleared too
        k_block_lists<<<num_batches, kUniqThreads, 0, s>>>(q);
        GC_CHECK_LAUNCH("gc_unique_compact lists");
        // ~8 CTAs per SM over the whole window
        unsigned gx = (unsigned)((sm_count() * 8u + num_batches - 1) / num_batches);
        if (gx < 1) gx = 1;
        const dim3 grid(gx, num_batches);
        k_block_counts<<<grid, kUniqThreads, 0, s>>>(q);
        GC_CHECK_LAUNCH("gc_unique_compact counts");
        k_block_scan<<<num_batches, 1024, 0, s>>>(q);
        GC_CHECK_LAUNCH("gc_unique_compact scan");
        k_block_emit<<<grid, kUniqThreads, 0, s>>>(q);
        GC_CHECK_LAUNCH("gc_unique_compact blocks");
        return GC_OK;
    }
    const unsigned tiles = uniq_tiles(visited);
    const uint32_t batch_ctas_from = g_unique_batch_min ? (uint32_t)g_unique_batch_min : sm_count();
    UniqueParams p{};
    p.bm = visited->bitmap;
    p.bwords = visited->words;
    p.tiles_per_batch = tiles;
    p.uniq = d_unique;
    p.ustride = unique_stride;
    p.ucount = d_unique_count;
    p.rank = reinterpret_cast<uint2*>(d_rank_table);
    p.feat = d_feat_lookups;
    p.clear = clear_bitmap;
    p.tile_count = static_cast<uint32_t*>(d_temp);
    if (num_batches >= batch_ctas_from) {
        k_unique_batch<<<num_batches, kFusedThreads, 0, s>>>(p);
        GC_CHECK_LAUNCH("gc_unique_compact batch");
        return GC_OK;
    }
    GC_REQUIRE(num_batches < 65536, GC_ERR_VALUE, "gc_unique_compact: at most 65535 batches per call");
    const dim3 grid(tiles, num_batches);
    k_unique_counts<<<grid, kUniqThreads, 0, s>>>(p);
    GC_CHECK_LAUNCH("gc_unique_compact counts");
    k_unique_tile_scan<<<num_batches, 1024, 0, s>>>(p);
    GC_CHECK_LAUNCH("gc_unique_compact scan");
    k_unique<<<grid, kUniqThreads, 0, s>>>(p);
    GC_CHECK_LAUNCH("gc_unique_compact");
    return GC_OK;
}

int gc_unique_compact_launches(uint32_t num_batches, const gc_visited_t* visited) {
    if (!visited || num_batches == 0) return 0;
    if (visited->summary) return 4;
    return num_batches >= (g_unique_batch_min ? (uint32_t)g_unique_batch_min : sm_count()) ? 1 : 3;
}

int gc_relabel(const uint32_t* d_ids, uint64_t ids_stride, const uint32_t* d_ids_count, uint32_t max_count,
               uint32_t num_batches, const uint32_t* d_rank_table, uint64_t bitmap_words, uint32_t* d_local,
               void* stream) {
    return relabel(d_ids, ids_stride, d_ids_count, max_count, num_batches, d_rank_table, bitmap_words, d_local, stream,
                   "gc_relabel");
}

int gc_relabel16(const uint32_t* d_ids, uint64_t ids_stride, const uint32_t* d_ids_count, uint32_t max_count,
                 uint32_t num_batches, const uint32_t* d_rank_table, uint64_t bitmap_words, uint16_t* d_local,
                 void* stream) {
    return relabel(d_ids, ids_stride, d_ids_count, max_count, num_batches, d_rank_table, bitmap_words, d_local, stream,
                   "gc_relabel16");
}

int gc_mark_visited(const uint32_t* d_ids, uint64_t ids_stride, const uint32_t* d_count, uint32_t max_count,
                    uint32_t num_batches, const gc_visited_t* visited, void* stream) {
    GC_REQUIRE(visited && visited->bitmap, GC_ERR_VALUE, "gc_mark_visited: visited set is null");
    GC_REQUIRE(num_batches < 65536, GC_ERR_VALUE, "gc_mark_visited: at most 65535 batches per call");
    if (num_batches == 0 || max_count == 0) return GC_OK;
    dim3 grid(grid_x(max_count, 256), num_batches);
    k_mark<<<grid, 256, 0, as_stream(stream)>>>(d_ids, ids_stride, d_count, visited->bitmap, visited->words,
                                                visited->summary, visited->summary_words);
    GC_CHECK_LAUNCH("gc_mark_visited");
    return GC_OK;
}

int gc_bitmap_clear(const gc_visited_t* visited, uint32_t num_batches, const uint32_t* d_unique,
                    uint64_t unique_stride, const uint32_t* d_unique_count, uint32_t max_unique, void* stream) {
    GC_REQUIRE(visited && visited->bitmap, GC_ERR_VALUE, "gc_bitmap_clear: visited set is null");
    GC_REQUIRE(num_batches < 65536, GC_ERR_VALUE, "gc_bitmap_clear: at most 65535 batches per call");
    if (num_batches == 0 || max_unique == 0) return GC_OK;
    dim3 grid(grid_x(max_unique, 256), num_batches);
    k_bitmap_clear<<<grid, 256, 0, as_stream(stream)>>>(visited->bitmap, visited->words, visited->summary,
                                                        visited->summary_words, d_unique, unique_stride,
                                                        d_unique_count);
    GC_CHECK_LAUNCH("gc_bitmap_clear");
    return GC_OK;
}

}  // extern "C"
