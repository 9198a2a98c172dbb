// K6/K7 cost-model kernels (planner.py:42-67, :87-121, :215-267):
//   colsum_argmax       clique-wide hotness totals and the first-argmax owner GPU
//   descending_order    CSLP ranking: totals descending, ties by ascending id — a
//                       hand-written stable LSD radix sort (8-bit digits of ~total,
//                       only as many passes as the largest total needs)
//   topo/hot prefix     inclusive byte and hotness scans along a ranking — a single-pass
//                       scan with decoupled look-back (gc_common.cuh)
//   searchsorted_right  batched boundary lookup for the alpha grid's float64 budgets
//   distribute_prefix   stable split of a ranked prefix into per-owner queues
// The final 101-point _estimate_at evaluation stays on the host, where Python's
// correctly rounded int/int division reproduces the reference bit for bit.
#include <cub/block/block_scan.cuh>

#include "gc_common.cuh"

namespace gc {

static unsigned grid1d(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
    return (unsigned)g;
}

__global__ void k_colsum_argmax(const int64_t* __restrict__ rows, uint32_t k, int64_t n, int64_t* __restrict__ totals,
                                int32_t* __restrict__ owner) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int64_t sum = 0, best = 0;
        int32_t arg = 0;
        for (uint32_t r = 0; r < k; ++r) {
            const int64_t x = rows[(int64_t)r * n + v];
            sum += x;
            if (r == 0 || x > best) {  // strict: first maximum wins (np.argmax)
                best = x;
                arg = (int32_t)r;
            }
        }
        if (totals) totals[v] = sum;
        if (owner) owner[v] = arg;
    }
}

__global__ void k_iota_keys(const int64_t* __restrict__ totals, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ ids, int64_t n) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        keys[v] = (uint64_t)totals[v];
        ids[v] = (uint32_t)v;
    }
}

__global__ void k_widen(const uint32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i];
}

__global__ void k_topo_cost(const uint64_t* __restrict__ ro, const int64_t* __restrict__ order, int64_t n,
                            uint32_t u32b, uint32_t u64b, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = order[i];
        out[i] = (int64_t)(ro[v + 1] - ro[v]) * u32b + u64b;
    }
}

__global__ void k_gather_i64(const int64_t* __restrict__ src, const int64_t* __restrict__ order, int64_t n,
                             int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = src[order[i]];
}

__global__ void k_searchsorted_right(const int64_t* __restrict__ prefix, int64_t n, const double* __restrict__ budgets,
                                     int32_t nb, int64_t* __restrict__ out) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb) return;
    const double b = budgets[i];
    int64_t lo = 0, hi = n;  // first index with (double)prefix[idx] > b
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if ((double)prefix[mid] <= b)
            lo = mid + 1;
        else
            hi = mid;
    }
    out[i] = lo;
}

// ---- stable multi-split by owner (distribute_prefix, planner.py:264-267)
constexpr int kSplitThreads = 256;
constexpr int kSplitRounds = 8;
constexpr int kSplitTile = kSplitThreads * kSplitRounds;

__global__ void k_split_count(const int64_t* __restrict__ order, int64_t len, const int32_t* __restrict__ owner,
                              uint32_t k, int64_t* __restrict__ tile_counts) {
    __shared__ unsigned s_cnt[GC_MAX_PEERS];
    if (threadIdx.x < GC_MAX_PEERS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSplitTile;
    for (int r = 0; r < kSplitRounds; ++r) {
        const int64_t i = base + r * kSplitThreads + threadIdx.x;
        if (i < len) atomicAdd(&s_cnt[owner[order[i]]], 1u);
    }
    __syncthreads();
    if (threadIdx.x < k) tile_counts[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s_cnt[threadIdx.x];
}

__global__ void k_split_place(const int64_t* __restrict__ order, int64_t len, const int32_t* __restrict__ owner,
                              uint32_t k, const int64_t* __restrict__ tile_offsets, int64_t* __restrict__ out) {
    __shared__ unsigned s_warp[kSplitThreads / 32][GC_MAX_PEERS];
    __shared__ int64_t s_run[GC_MAX_PEERS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < k) s_run[threadIdx.x] = tile_offsets[(int64_t)threadIdx.x * gridDim.x + blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kSplitTile;
    for (int r = 0; r < kSplitRounds; ++r) {
        const int64_t i = base + r * kSplitThreads + threadIdx.x;
        const bool valid = i < len;
        int64_t v = 0;
        int g = -1;
        if (valid) {
            v = order[i];
            g = owner[v];
        }
        unsigned my_rank = 0;
        for (uint32_t q = 0; q < k; ++q) {
            const unsigned m = __ballot_sync(kFull, g == (int)q);
            if (g == (int)q) my_rank = __popc(m & ((1u << lane) - 1u));
            if (lane == 0) s_warp[warp][q] = __popc(m);
        }
        __syncthreads();
        if (valid) {
            int64_t pos = s_run[g] + my_rank;
            for (int w = 0; w < warp; ++w) pos += s_warp[w][g];
            out[pos] = v;
        }
        __syncthreads();
        if (threadIdx.x < k) {
            int64_t add = 0;
            for (int w = 0; w < kSplitThreads / 32; ++w) add += s_warp[w][threadIdx.x];
            s_run[threadIdx.x] += add;
        }
        __syncthreads();
    }
}

// exclusive offsets in (owner-major, tile-minor) order + per-owner totals; one CTA
__global__ void __launch_bounds__(1024, 1) k_split_scan(const int64_t* __restrict__ tile_counts, int64_t tiles, uint32_t k,
                             int64_t* __restrict__ tile_offsets, int64_t* __restrict__ counts) {
    using Scan = cub::BlockScan<int64_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t g = 0; g < k; ++g) {
        const int64_t start_g = s_carry;
        for (int64_t t0 = 0; t0 < tiles; t0 += 1024) {
            const int64_t t = t0 + threadIdx.x;
            const int64_t c = t < tiles ? tile_counts[(int64_t)g * tiles + t] : 0;
            int64_t ex, agg;
            Scan(tmp).ExclusiveSum(c, ex, agg);
            if (t < tiles) tile_offsets[(int64_t)g * tiles + t] = s_carry + ex;
            __syncthreads();
            if (threadIdx.x == 0) s_carry += agg;
            __syncthreads();
        }
        if (threadIdx.x == 0) counts[g] = s_carry - start_g;
        __syncthreads();
    }
}

// ---- single-pass inclusive scan of non-negative int64 (decoupled look-back)
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

static int64_t scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }
static size_t scan_state_bytes(int64_t n) { return align_up((size_t)(scan_tiles(n) > 0 ? scan_tiles(n) : 1) * 8, 256) + 256; }

// in[] -> out[] (may alias). Tiles are claimed from `counter` (zeroed with `state`), so a
// tile's look-back only waits on tiles already held by running CTAs. `skip` (optional,
// device): the scan does nothing when *skip != 0 (inactive radix passes).
__global__ void __launch_bounds__(kScanThreads) k_scan_incl(const int64_t* in, int64_t n, int64_t* out,
                                                             uint64_t* __restrict__ state, uint32_t* __restrict__ counter,
                                                             const uint32_t* __restrict__ skip) {
    using BScan = cub::BlockScan<int64_t, kScanThreads>;
    __shared__ typename BScan::TempStorage tmp;
    __shared__ int64_t s_data[kScanTile];
    __shared__ uint32_t s_tile;
    __shared__ int64_t s_prefix;
    if (skip && *skip) return;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * kScanTile;
#pragma unroll
    for (int r = 0; r < kScanItems; ++r) {  // coalesced, striped
        const int64_t i = base + r * kScanThreads + tid;
        s_data[r * kScanThreads + tid] = i < n ? in[i] : 0;
    }
    __syncthreads();
    int64_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) sum += s_data[tid * kScanItems + k];  // blocked
    int64_t excl, total;
    BScan(tmp).ExclusiveSum(sum, excl, total);
    // the aggregate first, so successors sum past this tile instead of waiting for its prefix
    if (tid == 0 && tile != 0) publish(state + tile, kFlagAgg | (uint64_t)total);
    if (tid < 32) {
        const uint64_t pre = lookback_warp(state, 0, tile, (uint64_t)total);
        if ((tid & 31) == 0) s_prefix = (int64_t)pre;
    }
    __syncthreads();
    int64_t run = s_prefix + excl;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        run += s_data[tid * kScanItems + k];
        s_data[tid * kScanItems + k] = run;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kScanItems; ++r) {
        const int64_t i = base + r * kScanThreads + tid;
        if (i < n) out[i] = s_data[r * kScanThreads + tid];
    }
}

static int scan_incl(const int64_t* in, int64_t n, int64_t* out, void* state_buf, cudaStream_t s,
                     const uint32_t* skip, const char* what) {
    const int64_t tiles = scan_tiles(n);
    GC_REQUIRE(tiles < (1ll << 31), GC_ERR_VALUE, "scan: too many items");
    const size_t sb = scan_state_bytes(n);
    GC_TRY(cudaMemsetAsync(state_buf, 0, sb, s), what);
    auto* state = static_cast<uint64_t*>(state_buf);
    auto* counter = reinterpret_cast<uint32_t*>(static_cast<char*>(state_buf) + sb - 256);
    k_scan_incl<<<(unsigned)(tiles > 0 ? tiles : 1), kScanThreads, 0, s>>>(in, n, out, state, counter, skip);
    GC_CHECK_LAUNCH(what);
    return GC_OK;
}

// ---- stable LSD radix sort of (~key, id): descending keys, equal keys by ascending id
constexpr int kRadixThreads = 256;
constexpr int kRadixRounds = 16;
constexpr int kRadixTile = kRadixThreads * kRadixRounds;
constexpr int kRadixBins = 256;
constexpr int kRadixPasses = 8;  // 64-bit keys; passes above the largest key's top bit do nothing

static int64_t radix_tiles(int64_t n) { return (n + kRadixTile - 1) / kRadixTile; }

__device__ __forceinline__ uint32_t desc_digit(uint64_t key, int pass) { return 255u - (uint32_t)((key >> (8 * pass)) & 0xFFu); }

// bits[0] = significant bits of the largest key; bits[1 + p] = 1 if pass p is skipped
__global__ void k_radix_bits(const uint64_t* __restrict__ maxkey, uint32_t* __restrict__ bits) {
    if (threadIdx.x == 0) {
        const uint64_t m = *maxkey;
        const uint32_t b = m ? 64u - (uint32_t)__clzll((long long)m) : 0u;
        bits[0] = b;
        for (int p = 0; p < kRadixPasses; ++p) bits[1 + p] = (uint32_t)(8 * p) >= b;
    }
}

__global__ void k_max_u64(const uint64_t* __restrict__ keys, int64_t n, unsigned long long* __restrict__ out) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (unsigned long long)keys[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// per-tile digit counts, digit-major: hist[d * tiles + tile]
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const uint64_t* __restrict__ keys, int64_t n, int pass,
                                                               const uint32_t* __restrict__ bits,
                                                               int64_t* __restrict__ hist) {
    __shared__ uint32_t s_cnt[kRadixBins];
    if (bits[1 + pass]) return;
    const int tid = threadIdx.x, lane = tid & 31;
    s_cnt[tid] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRadixTile;
    for (int r = 0; r < kRadixRounds; ++r) {
        const int64_t i = base + r * kRadixThreads + tid;
        const bool valid = i < n;
        const uint32_t d = valid ? desc_digit(keys[i], pass) : 0u;
        // one shared atomic per distinct digit per warp (zero hotness fills most bins' peers)
        const unsigned act = __ballot_sync(kFull, valid);
        if (valid) {
            const unsigned peers = __match_any_sync(act, d);
            if (lane == __ffs(peers) - 1) atomicAdd(&s_cnt[d], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    hist[(int64_t)tid * gridDim.x + blockIdx.x] = s_cnt[tid];
}

// stable scatter: items keep their index order within a digit (round, then warp, then lane)
__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(const uint64_t* __restrict__ kin,
                                                                  const uint32_t* __restrict__ vin, int64_t n, int pass,
                                                                  const uint32_t* __restrict__ bits,
                                                                  const int64_t* __restrict__ hist,
                                                                  const int64_t* __restrict__ incl,
                                                                  uint64_t* __restrict__ kout,
                                                                  uint32_t* __restrict__ vout) {
    constexpr int kWarps = kRadixThreads / 32;
    __shared__ int64_t s_run[kRadixBins];
    __shared__ uint32_t s_wcnt[kWarps][kRadixBins];
    if (bits[1 + pass]) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {
        const int64_t h = (int64_t)tid * gridDim.x + blockIdx.x;
        s_run[tid] = incl[h] - hist[h];  // exclusive offset of (digit tid, this tile)
    }
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s_wcnt[w][tid] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRadixTile;
    for (int r = 0; r < kRadixRounds; ++r) {
        const int64_t i = base + r * kRadixThreads + tid;
        const bool valid = i < n;
        uint64_t key = 0;
        uint32_t val = 0, d = 0, rank = 0;
        const unsigned act = __ballot_sync(kFull, valid);
        if (valid) {
            key = kin[i];
            val = vin[i];
            d = desc_digit(key, pass);
            const unsigned peers = __match_any_sync(act, d);
            rank = __popc(peers & ((1u << lane) - 1u));
            if (lane == __ffs(peers) - 1) s_wcnt[warp][d] = (uint32_t)__popc(peers);
        }
        __syncthreads();
        if (valid) {
            int64_t pos = s_run[d] + rank;
            for (int w = 0; w < warp; ++w) pos += s_wcnt[w][d];
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
        {
            uint32_t add = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                add += s_wcnt[w][tid];
                s_wcnt[w][tid] = 0;
            }
            s_run[tid] += add;
        }
        __syncthreads();
    }
}

// the sorted ids are in v0 after an even number of executed passes, else in v1
__global__ void k_widen_sorted(const uint32_t* __restrict__ v0, const uint32_t* __restrict__ v1,
                               const uint32_t* __restrict__ bits, int64_t n, int64_t* __restrict__ out) {
    const uint32_t passes = (bits[0] + 7) / 8;
    const uint32_t* in = (passes & 1u) ? v1 : v0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i];
}

struct SortLayout {
    size_t k0, k1, v0, v1, hist, incl, state, misc, total;
};

static SortLayout sort_layout(int64_t n) {
    SortLayout L{};
    const int64_t nh = (int64_t)kRadixBins * (radix_tiles(n) > 0 ? radix_tiles(n) : 1);
    size_t off = 0;
    L.k0 = off; off = align_up(off + 8 * (size_t)n, 256);
    L.k1 = off; off = align_up(off + 8 * (size_t)n, 256);
    L.v0 = off; off = align_up(off + 4 * (size_t)n, 256);
    L.v1 = off; off = align_up(off + 4 * (size_t)n, 256);
    L.hist = off; off = align_up(off + 8 * (size_t)nh, 256);
    L.incl = off; off = align_up(off + 8 * (size_t)nh, 256);
    L.state = off; off = align_up(off + scan_state_bytes(nh), 256);
    L.misc = off; off = align_up(off + 256, 256);  // max key (u64) + pass flags (u32[1 + passes])
    L.total = off;
    return L;
}

}  // namespace gc

using namespace gc;

extern "C" {

int gc_colsum_argmax(const int64_t* d_rows, uint32_t k_rows, int64_t n, int64_t* d_totals, int32_t* d_owner,
                     void* stream) {
    GC_REQUIRE(k_rows >= 1 && n >= 0, GC_ERR_VALUE, "gc_colsum_argmax: need k_rows >= 1, n >= 0");
    if (n == 0) return GC_OK;
    k_colsum_argmax<<<grid1d(n, 256), 256, 0, as_stream(stream)>>>(d_rows, k_rows, n, d_totals, d_owner);
    GC_CHECK_LAUNCH("gc_colsum_argmax");
    return GC_OK;
}

size_t gc_descending_order_temp_bytes(int64_t n) { return n < 0 ? 0 : sort_layout(n).total; }

int gc_descending_order(const int64_t* d_totals, int64_t n, int64_t* d_order, void* d_temp, size_t temp_bytes,
                        void* stream) {
    GC_REQUIRE(n >= 0 && n < (1ll << 31), GC_ERR_VALUE, "gc_descending_order: n must be in [0, 2^31)");
    if (n == 0) return GC_OK;
    SortLayout L = sort_layout(n);
    GC_REQUIRE(d_temp && temp_bytes >= L.total, GC_ERR_VALUE, "gc_descending_order: temp buffer too small");
    char* t = static_cast<char*>(d_temp);
    cudaStream_t s = as_stream(stream);
    auto* k0 = reinterpret_cast<uint64_t*>(t + L.k0);
    auto* k1 = reinterpret_cast<uint64_t*>(t + L.k1);
    auto* v0 = reinterpret_cast<uint32_t*>(t + L.v0);
    auto* v1 = reinterpret_cast<uint32_t*>(t + L.v1);
    k_iota_keys<<<grid1d(n, 256), 256, 0, s>>>(d_totals, k0, v0, n);
    GC_CHECK_LAUNCH("gc_descending_order keys");
    // stable descending radix sort: equal totals keep ascending id, which is the
    // lexsort((arange(n), -totals)) order of planner.py:45
    auto* maxkey = reinterpret_cast<unsigned long long*>(t + L.misc);
    auto* bits = reinterpret_cast<uint32_t*>(t + L.misc + 8);
    GC_TRY(cudaMemsetAsync(maxkey, 0, 8, s), "gc_descending_order memset");
    k_max_u64<<<grid1d(n, 256), 256, 0, s>>>(k0, n, maxkey);
    k_radix_bits<<<1, 32, 0, s>>>(reinterpret_cast<const uint64_t*>(maxkey), bits);
    GC_CHECK_LAUNCH("gc_descending_order max");
    const int64_t tiles = radix_tiles(n);
    GC_REQUIRE(tiles < (1ll << 31), GC_ERR_VALUE, "gc_descending_order: too many items");
    const int64_t nh = (int64_t)kRadixBins * tiles;
    auto* hist = reinterpret_cast<int64_t*>(t + L.hist);
    auto* incl = reinterpret_cast<int64_t*>(t + L.incl);
    uint64_t* kb[2] = {k0, k1};
    uint32_t* vb[2] = {v0, v1};
    // pass p reads buffer p & 1 when every earlier pass ran; a skipped pass implies all
    // later ones skip too (their digits are zero), so the parity stays consistent
    for (int p = 0; p < kRadixPasses; ++p) {
        k_radix_hist<<<(unsigned)tiles, kRadixThreads, 0, s>>>(kb[p & 1], n, p, bits, hist);
        GC_CHECK_LAUNCH("gc_descending_order hist");
        const int rc = scan_incl(hist, nh, incl, t + L.state, s, bits + 1 + p, "gc_descending_order scan");
        if (rc != GC_OK) return rc;
        k_radix_scatter<<<(unsigned)tiles, kRadixThreads, 0, s>>>(kb[p & 1], vb[p & 1], n, p, bits, hist, incl,
                                                                  kb[(p + 1) & 1], vb[(p + 1) & 1]);
        GC_CHECK_LAUNCH("gc_descending_order scatter");
    }
    k_widen_sorted<<<grid1d(n, 256), 256, 0, s>>>(v0, v1, bits, n, d_order);
    GC_CHECK_LAUNCH("gc_descending_order widen");
    return GC_OK;
}

size_t gc_order_scan_temp_bytes(int64_t n) {
    if (n < 0) return 0;
    return align_up(8 * (size_t)n, 256) + scan_state_bytes(n);
}

static int order_scan(const int64_t* vals, int64_t n, int64_t* d_out, void* d_temp, size_t temp_bytes, cudaStream_t s,
                      const char* what) {
    (void)temp_bytes;
    return scan_incl(vals, n, d_out, static_cast<char*>(d_temp) + align_up(8 * (size_t)n, 256), s, nullptr, what);
}

int gc_topo_prefix_bytes(const uint64_t* d_row_offsets, const int64_t* d_order, int64_t n, uint32_t u32_bytes,
                         uint32_t u64_bytes, int64_t* d_out, void* d_temp, size_t temp_bytes, void* stream) {
    GC_REQUIRE(n >= 0 && n < (1ll << 31), GC_ERR_VALUE, "gc_topo_prefix_bytes: n must be in [0, 2^31)");
    if (n == 0) return GC_OK;
    GC_REQUIRE(d_temp && temp_bytes >= gc_order_scan_temp_bytes(n), GC_ERR_VALUE,
               "gc_topo_prefix_bytes: temp buffer too small");
    cudaStream_t s = as_stream(stream);
    auto* vals = static_cast<int64_t*>(d_temp);
    k_topo_cost<<<grid1d(n, 256), 256, 0, s>>>(d_row_offsets, d_order, n, u32_bytes, u64_bytes, vals);
    GC_CHECK_LAUNCH("gc_topo_prefix_bytes");
    return order_scan(vals, n, d_out, d_temp, temp_bytes, s, "gc_topo_prefix_bytes scan");
}

int gc_hot_prefix(const int64_t* d_totals, const int64_t* d_order, int64_t n, int64_t* d_out, void* d_temp,
                  size_t temp_bytes, void* stream) {
    GC_REQUIRE(n >= 0 && n < (1ll << 31), GC_ERR_VALUE, "gc_hot_prefix: n must be in [0, 2^31)");
    if (n == 0) return GC_OK;
    GC_REQUIRE(d_temp && temp_bytes >= gc_order_scan_temp_bytes(n), GC_ERR_VALUE,
               "gc_hot_prefix: temp buffer too small");
    cudaStream_t s = as_stream(stream);
    auto* vals = static_cast<int64_t*>(d_temp);
    k_gather_i64<<<grid1d(n, 256), 256, 0, s>>>(d_totals, d_order, n, vals);
    GC_CHECK_LAUNCH("gc_hot_prefix");
    return order_scan(vals, n, d_out, d_temp, temp_bytes, s, "gc_hot_prefix scan");
}

int gc_searchsorted_right(const int64_t* d_prefix, int64_t n, const double* d_budgets, int32_t num_budgets,
                          int64_t* d_out, void* stream) {
    GC_REQUIRE(n >= 0 && num_budgets >= 0, GC_ERR_VALUE, "gc_searchsorted_right: negative size");
    if (num_budgets == 0) return GC_OK;
    k_searchsorted_right<<<(num_budgets + 127) / 128, 128, 0, as_stream(stream)>>>(d_prefix, n, d_budgets,
                                                                                  num_budgets, d_out);
    GC_CHECK_LAUNCH("gc_searchsorted_right");
    return GC_OK;
}

size_t gc_distribute_prefix_temp_bytes(int64_t len, uint32_t k_rows) {
    const int64_t tiles = (len + kSplitTile - 1) / kSplitTile;
    return 2 * align_up((size_t)(tiles > 0 ? tiles : 1) * k_rows * 8, 256);
}

int gc_distribute_prefix(const int64_t* d_order, int64_t len, const int32_t* d_owner, uint32_t k_rows, int64_t* d_out,
                         int64_t* d_counts, void* d_temp, size_t temp_bytes, void* stream) {
    GC_REQUIRE(k_rows >= 1 && k_rows <= GC_MAX_PEERS, GC_ERR_VALUE, "gc_distribute_prefix: 1 <= k_rows <= 8");
    GC_REQUIRE(len >= 0, GC_ERR_VALUE, "gc_distribute_prefix: len must be >= 0");
    cudaStream_t s = as_stream(stream);
    if (len == 0) {
        GC_TRY(cudaMemsetAsync(d_counts, 0, 8 * k_rows, s), "gc_distribute_prefix memset");
        return GC_OK;
    }
    GC_REQUIRE(d_temp && temp_bytes >= gc_distribute_prefix_temp_bytes(len, k_rows), GC_ERR_VALUE,
               "gc_distribute_prefix: temp buffer too small");
    const int64_t tiles = (len + kSplitTile - 1) / kSplitTile;
    GC_REQUIRE(tiles < (1ll << 31), GC_ERR_VALUE, "gc_distribute_prefix: too many items");
    auto* tile_counts = static_cast<int64_t*>(d_temp);
    auto* tile_offsets =
        reinterpret_cast<int64_t*>(static_cast<char*>(d_temp) + align_up((size_t)tiles * k_rows * 8, 256));
    k_split_count<<<(unsigned)tiles, kSplitThreads, 0, s>>>(d_order, len, d_owner, k_rows, tile_counts);
    GC_CHECK_LAUNCH("gc_distribute_prefix count");
    k_split_scan<<<1, 1024, 0, s>>>(tile_counts, tiles, k_rows, tile_offsets, d_counts);
    GC_CHECK_LAUNCH("gc_distribute_prefix scan");
    k_split_place<<<(unsigned)tiles, kSplitThreads, 0, s>>>(d_order, len, d_owner, k_rows, tile_offsets, d_out);
    GC_CHECK_LAUNCH("gc_distribute_prefix place");
    return GC_OK;
}

}  // extern "C"
