// K4 gather3tier + K5 hotness scatter.
//
// gather: every distinct vertex of a batch gets its feature row from the tier that
// holds it (the serving rule of account_assignment, simulator.py:161-202):
//   local HBM slab, an NVLink/NVSwitch peer's slab (one-sided loads through a mapped
//   peer pointer; the owner is the unique holder CSLP assigned, planner.py:54-55), or
//   the host feature table over PCIe through a UVA pointer to mapped pinned memory.
// Rows move as 16-byte vectors with one thread per vector, so a warp covers
// contiguous output and each row's source bytes are read once, fully coalesced.
#include "gc_common.cuh"

#ifndef GC_GATHER_MIN_BLOCKS
#define GC_GATHER_MIN_BLOCKS 6  // 40 registers: 48 warps per SM (C2 gather 0.527 -> 0.466 ms)
#endif
#ifndef GC_GATHER_ROWS
#define GC_GATHER_ROWS 4  // rows in flight per warp in k_gather_rows
#endif

namespace gc {

// deferred host-tier row: destination row index in `out` and the vertex id
struct DeferredRow {
    uint64_t dst_row;
    uint32_t id;
    uint32_t pad;
};

struct GatherParams {
    gc_feature_store_t fs;
    DeferredRow* defer;  // non-null: host-tier rows are listed here instead of read
    uint32_t* defer_count;
    const uint32_t* ids;
    uint64_t ids_stride;
    const uint32_t* count;
    char* out;
    uint64_t out_stride_rows;
    uint64_t* tier_rows;
    uint32_t max_rows;
};

__device__ __forceinline__ uint4 ld_stream16(const void* ptr) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr));
    return r;
}

__device__ __forceinline__ void st_stream16(void* ptr, uint4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// tier: 0 local, 1 peer, 2 host
__device__ __forceinline__ const char* row_source(const gc_feature_store_t& fs, uint32_t u, int& tier) {
    if (fs.location == nullptr) {
        tier = 0;
        return static_cast<const char*>(fs.slabs[fs.self_rank]) + (uint64_t)u * fs.row_bytes;
    }
    const uint32_t loc = __ldg(fs.location + u);
    if (loc == GC_TIER_HOST) {
        tier = 2;
        return static_cast<const char*>(fs.host_rows) + (uint64_t)u * fs.row_bytes;
    }
    const uint32_t g = loc >> 28;
    tier = (g == fs.self_rank) ? 0 : 1;
    return static_cast<const char*>(fs.slabs[g]) + (uint64_t)(loc & 0x0FFFFFFFu) * fs.row_bytes;
}

template <int VEC>
__global__ void __launch_bounds__(256) k_gather(GatherParams p) {
    __shared__ unsigned long long s_tier[3];
    const uint32_t b = blockIdx.y;
    const uint32_t rows = min(p.count[b], p.max_rows);  // capacity clamp; caller checks overflow
    const uint32_t per_row = p.fs.row_bytes / VEC;
    const uint64_t total = (uint64_t)rows * per_row;
    const uint32_t* ids = p.ids + b * p.ids_stride;
    char* out = p.out + b * p.out_stride_rows * p.fs.row_bytes;
    if (p.tier_rows && threadIdx.x < 3) s_tier[threadIdx.x] = 0;
    if (p.tier_rows) __syncthreads();
    unsigned long long cnt[3] = {0, 0, 0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = (uint32_t)(i / per_row);
        const uint32_t c = (uint32_t)(i - (uint64_t)k * per_row);
        int tier;
        const char* src = row_source(p.fs, __ldg(ids + k), tier) + (uint64_t)c * VEC;
        char* dst = out + (uint64_t)k * p.fs.row_bytes + (uint64_t)c * VEC;
        if constexpr (VEC == 16) {
            st_stream16(dst, ld_stream16(src));
        } else {
            *reinterpret_cast<uint32_t*>(dst) = __ldg(reinterpret_cast<const uint32_t*>(src));
        }
        if (c == 0) {
            cnt[0] += tier == 0;
            cnt[1] += tier == 1;
            cnt[2] += tier == 2;
        }
    }
    if (p.tier_rows) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            unsigned long long v = cnt[t];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_tier[t], v);
        }
        __syncthreads();
        if (threadIdx.x < 3 && s_tier[threadIdx.x])
            atomicAdd((unsigned long long*)(p.tier_rows + threadIdx.x), s_tier[threadIdx.x]);
    }
}

// Warp-per-row gather for 16-byte-aligned rows of at most 32*VPL vectors (VPL = 1:
// D <= 128 fp32; 2: D <= 256, C5's 1024-byte rows; 4: D <= 512): lane l moves vectors
// l, l+32, ... of a row. Each warp keeps ROWS rows in flight — their ids and
// locations are fetched by ROWS lanes at once and broadcast, then ROWS independent
// 16-byte loads per lane are issued before any store — so HBM, NVLink and PCIe
// latency overlap instead of serialising per row.
template <int ROWS, int VPL>
__global__ void __launch_bounds__(256, VPL == 1 ? GC_GATHER_MIN_BLOCKS : 4) k_gather_rows(GatherParams p) {
    __shared__ unsigned long long s_tier[3];
    const uint32_t b = blockIdx.y;
    const uint32_t rows = min(p.count[b], p.max_rows);
    const uint32_t per_row = p.fs.row_bytes / 16;  // <= 32 * VPL
    const uint32_t* ids = p.ids + b * p.ids_stride;
    char* out = p.out + b * p.out_stride_rows * p.fs.row_bytes;
    const int lane = threadIdx.x & 31;
    if (p.tier_rows && threadIdx.x < 3) s_tier[threadIdx.x] = 0;
    if (p.tier_rows) __syncthreads();
    unsigned long long cnt[3] = {0, 0, 0};
    const uint32_t warps = gridDim.x * (blockDim.x / 32);
    const uint32_t wid = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    // each warp takes 32 consecutive rows: one coalesced id load and one location
    // lookup per lane resolve all 32 sources, then ROWS rows at a time move with
    // ROWS independent 16-byte loads per lane in flight before their stores
    for (uint32_t c0 = wid * 32; c0 < rows; c0 += warps * 32) {
        const char* my_src = nullptr;
        int my_tier = 0;
        uint32_t my_id = 0;
        if (c0 + lane < rows) {
            my_id = __ldg(ids + c0 + lane);
            my_src = row_source(p.fs, my_id, my_tier);
            cnt[0] += my_tier == 0;
            cnt[1] += my_tier == 1;
            cnt[2] += my_tier == 2;
        }
        if (p.defer) {
            // host rows go to the deferred list (read later by a few warps over PCIe);
            // one atomic per warp, plus the largest listed id (the address sort's range)
            const bool d = my_src != nullptr && my_tier == 2;
            const unsigned m = __ballot_sync(kFull, d);
            if (m) {
                uint32_t base = 0;
                const uint32_t mx = __reduce_max_sync(kFull, d ? my_id : 0u);
                if (lane == __ffs(m) - 1) {
                    base = atomicAdd(p.defer_count, (uint32_t)__popc(m));
                    atomicMax(p.defer_count + 1, mx);
                }
                base = __shfl_sync(kFull, base, __ffs(m) - 1);
                if (d) {
                    DeferredRow e;
                    e.dst_row = (uint64_t)b * p.out_stride_rows + c0 + lane;
                    e.id = my_id;
                    e.pad = 0;
                    p.defer[base + __popc(m & ((1u << lane) - 1u))] = e;
                    my_src = nullptr;
                }
            }
        }
        const uint32_t n = min(32u, rows - c0);
        if constexpr (VPL == 1) {
            for (uint32_t j0 = 0; j0 < n; j0 += ROWS) {
                uint4 v[ROWS];
#pragma unroll
                for (int j = 0; j < ROWS; ++j) {
                    const char* src = (const char*)__shfl_sync(kFull, (unsigned long long)my_src, (j0 + j) & 31);
                    v[j] = (j0 + j < n && src && (uint32_t)lane < per_row) ? ld_stream16(src + 16 * lane)
                                                                             : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int j = 0; j < ROWS; ++j) {
                    const bool have = __shfl_sync(kFull, my_src != nullptr, (j0 + j) & 31);
                    if (j0 + j < n && have && (uint32_t)lane < per_row)
                        st_stream16(out + (uint64_t)(c0 + j0 + j) * p.fs.row_bytes + 16 * lane, v[j]);
                }
            }
            continue;
        }
        for (uint32_t j0 = 0; j0 < n; j0 += ROWS) {
            uint4 v[ROWS][VPL];
#pragma unroll
            for (int j = 0; j < ROWS; ++j) {
                const char* src = (const char*)__shfl_sync(kFull, (unsigned long long)my_src, (j0 + j) & 31);
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    const uint32_t c = (uint32_t)lane + 32u * q;
                    v[j][q] = (j0 + j < n && src && c < per_row) ? ld_stream16(src + 16 * c) : make_uint4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int j = 0; j < ROWS; ++j) {
                const bool have = __shfl_sync(kFull, my_src != nullptr, (j0 + j) & 31);
                char* dst = out + (uint64_t)(c0 + j0 + j) * p.fs.row_bytes;
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    const uint32_t c = (uint32_t)lane + 32u * q;
                    if (j0 + j < n && have && c < per_row) st_stream16(dst + 16 * c, v[j][q]);
                }
            }
        }
    }
    if (p.tier_rows) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            unsigned long long v = cnt[t];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_tier[t], v);
        }
        __syncthreads();
        if (threadIdx.x < 3 && s_tier[threadIdx.x])
            atomicAdd((unsigned long long*)(p.tier_rows + threadIdx.x), s_tier[threadIdx.x]);
    }
}

// host-row kernel grid (GC_OPT_DEFER_CTAS): 2 CTAs per SM of one warp and ~33 KB of
// shared memory each, so they fit beside the sampling kernels
static int g_defer_ctas = 296;
void set_defer_ctas(int ctas) { g_defer_ctas = ctas; }
// warp-per-row gather grid: CTAs per SM over the whole window (16 fills the GPU; fewer
// leave room for another lane's kernels while a PCIe-bound gather runs)
static int g_gather_ctas_per_sm = 16;
void set_gather_ctas_per_sm(int v) { g_gather_ctas_per_sm = v; }

// Deferred host-tier rows by TMA bulk copies: a 32-thread CTA stages up to R list
// entries in shared memory, then one lane issues R cp.async.bulk reads of whole rows
// from the pinned host table (UVA; completion counted on one mbarrier per row) and, as
// each lands, a bulk write of the row to its destination. R rows (32 KB) stay in flight
// per CTA while the CTA holds one warp's issue slots and no registers to speak of, so
// the PCIe-latency-bound reads leave the SMs to the next window's sampling kernels.
// (tools/tma_host_probe.cu: one such CTA per SM reaches the box's host-read limit.)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) k_gather_deferred_tma(const char* __restrict__ host_rows, uint32_t row_bytes,
                                                            const DeferredRow* __restrict__ list,
                                                            const uint32_t* __restrict__ count, char* out, int R) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);          // [R] mbarriers
    uint64_t* src = bar + R;                                     // [R] host byte offsets
    uint64_t* dst = src + R;                                     // [R] destination rows
    char* buf = reinterpret_cast<char*>(smem) + ((size_t)24 * R + 127) / 128 * 128;  // [R][row_bytes]
    const uint32_t n = *count;
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int k = 0; k < R; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[k])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase = 0;
    for (uint32_t r0 = blockIdx.x * (uint32_t)R; r0 < n; r0 += gridDim.x * (uint32_t)R) {
        const uint32_t m = min((uint32_t)R, n - r0);
        for (uint32_t k = lane; k < m; k += 32) {
            const DeferredRow e = list[r0 + k];
            src[k] = (uint64_t)e.id * row_bytes;
            dst[k] = e.dst_row;
        }
        __syncwarp();
        if (lane == 0) {
            for (uint32_t k = 0; k < m; ++k) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[k])),
                             "r"(row_bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_addr(buf + (size_t)k * row_bytes)),
                    "l"(host_rows + src[k]), "r"(row_bytes), "r"(smem_addr(&bar[k]))
                    : "memory");
            }
            for (uint32_t k = 0; k < m; ++k) {
                uint32_t done = 0;
                while (!done)
                    asm volatile(
                        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                        : "=r"(done)
                        : "r"(smem_addr(&bar[k])), "r"(phase)
                        : "memory");
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                 out + dst[k] * row_bytes),
                             "r"(smem_addr(buf + (size_t)k * row_bytes)), "r"(row_bytes)
                             : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the buffers may be refilled
        }
        phase ^= 1u;  // only the CTA's last round can be partial
        __syncwarp();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes complete before exit
}

// Address order for the deferred host rows (GC_OPT_DEFER_ORDER = 1). Random 512-byte
// reads from a 56 GiB pinned table reach 26 GB/s on the B200 box, the same ids issued in
// ascending order 41 GB/s (tools/host_page_probe.py, profiles/r02_host_tier_pages.md):
// the host-side address translation, not the link, limits random reads. So the window's
// list is bucket-sorted by id (65536 buckets over [0, max id]: histogram, one-CTA scan,
// scatter) before the TMA kernel walks it; CTAs claim consecutive runs, so the reads in
// flight at any moment cover a narrow address range. Order within a bucket is free:
// every entry names its destination row, so the output does not depend on it.
constexpr uint32_t kDeferBuckets = 1u << 16;
static int g_defer_order = 1;
void set_defer_order(int v) { g_defer_order = v; }

__device__ __forceinline__ uint32_t defer_shift(const uint32_t* hdr) {
    const int bits = 32 - __clz(hdr[1] | 1u);
    return bits > 16 ? (uint32_t)(bits - 16) : 0u;
}

__global__ void __launch_bounds__(256) k_defer_hist(const DeferredRow* __restrict__ list, const uint32_t* hdr,
                                                    uint32_t* __restrict__ hist) {
    const uint32_t n = hdr[0], sh = defer_shift(hdr);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&hist[list[i].id >> sh], 1u);
}

// exclusive scan of the 65536 bucket counts in place: 1024 threads x 64 counts
static_assert(kDeferBuckets == 1024u * 64u, "k_defer_scan covers 1024 x 64 buckets");
__global__ void __launch_bounds__(1024) k_defer_scan(uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_sum[1024];
    const uint32_t t = threadIdx.x;
    uint4* h = reinterpret_cast<uint4*>(hist + t * 64);
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint4 v = h[k];
        sum += v.x + v.y + v.z + v.w;
    }
    s_sum[t] = sum;
    __syncthreads();
    for (uint32_t o = 1; o < 1024; o <<= 1) {
        const uint32_t v = t >= o ? s_sum[t - o] : 0u;
        __syncthreads();
        s_sum[t] += v;
        __syncthreads();
    }
    uint32_t run = s_sum[t] - sum;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        uint4 v = h[k];
        const uint4 c = v;
        v.x = run;
        v.y = v.x + c.x;
        v.z = v.y + c.y;
        v.w = v.z + c.z;
        run = v.w + c.w;
        h[k] = v;
    }
}

__global__ void __launch_bounds__(256) k_defer_scatter(const DeferredRow* __restrict__ list, const uint32_t* hdr,
                                                       uint32_t* __restrict__ cursor, DeferredRow* __restrict__ sorted) {
    const uint32_t n = hdr[0], sh = defer_shift(hdr);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const DeferredRow e = list[i];
        sorted[atomicAdd(&cursor[e.id >> sh], 1u)] = e;
    }
}

// rows in flight per host-row CTA: 0 = ~32 KB of rows (at most 64); otherwise the
// GC_OPT_DEFER_ROWS value (a few fat CTAs — e.g. 16 x 384 rows — hold only a few SMs'
// shared memory, leaving the rest to the next window's sampling)
static int g_defer_rows = 0;
void set_defer_rows(int v) { g_defer_rows = v; }

static int defer_rows_in_flight(uint32_t row_bytes) {
    if (g_defer_rows > 0) return g_defer_rows;
    int r = (int)(32768u / row_bytes);
    return r > 64 ? 64 : (r < 1 ? 1 : r);
}

// accumulate_hotness bincount (sampling.py:171-173) with warp aggregation for hot ids
__global__ void k_scatter_add(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ w, int64_t n,
                              uint64_t* counter) {
    const int lane = threadIdx.x & 31;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const uint32_t u = valid ? ids[i] : 0u;
        const uint64_t add = valid ? (w ? (uint64_t)w[i] : 1ull) : 0ull;
        const unsigned act = __ballot_sync(kFull, valid);
        if (valid) {
            const unsigned peers = __match_any_sync(act, u);
            // segmented sum over the peer group through shuffles
            uint64_t sum = 0;
            unsigned rem = peers;
            while (rem) {
                const int src = __ffs(rem) - 1;
                sum += __shfl_sync(peers, add, src);
                rem &= rem - 1;
            }
            if (lane == __ffs(peers) - 1 && sum) atomicAdd((unsigned long long*)(counter + u), (unsigned long long)sum);
        }
    }
}

// Deterministic synthetic feature table (bench/test input, identical to the CPU
// restatement in oracle/): X[v, d] = (mix64(v*D + d) >> 40) * 2^-24 - 0.5, exact in fp32.
__global__ void k_synth_features(uint64_t first_row, uint64_t rows, uint32_t dim, float* __restrict__ out) {
    const uint64_t total = rows * dim;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = first_row + i / dim;
        const uint64_t d = i % dim;
        out[i] = (float)(mix64(v * dim + d) >> 40) * (1.0f / 16777216.0f) - 0.5f;
    }
}

}  // namespace gc

using namespace gc;

extern "C" {

uint64_t gc_gather_defer_bytes(uint32_t max_count, uint32_t num_batches);

static int gather_impl(const gc_feature_store_t* store, const uint32_t* d_ids, uint64_t ids_stride,
                       const uint32_t* d_count, uint32_t max_count, uint32_t num_batches, void* d_out,
                       uint64_t out_stride_rows, uint64_t* d_tier_rows, void* d_defer, uint64_t defer_bytes,
                       void* stream, void* host_stream) {
    GC_REQUIRE(store, GC_ERR_VALUE, "gc_gather: store is null");
    GC_REQUIRE(store->row_bytes > 0 && store->row_bytes % 4 == 0, GC_ERR_VALUE,
               "gc_gather: row_bytes must be a positive multiple of 4");
    GC_REQUIRE(store->self_rank < GC_MAX_PEERS, GC_ERR_VALUE, "gc_gather: self_rank out of range");
    GC_REQUIRE(num_batches < 65536, GC_ERR_VALUE, "gc_gather: at most 65535 batches per call");
    if (num_batches == 0 || max_count == 0) return GC_OK;
    GatherParams p{};
    p.fs = *store;
    p.ids = d_ids;
    p.ids_stride = ids_stride;
    p.count = d_count;
    p.out = static_cast<char*>(d_out);
    p.out_stride_rows = out_stride_rows;
    p.tier_rows = d_tier_rows;
    p.max_rows = max_count;
    const bool vec16 = store->row_bytes % 16 == 0 && ((uintptr_t)d_out % 16 == 0);
    const uint32_t per_row = store->row_bytes / (vec16 ? 16 : 4);
    cudaStream_t s = as_stream(stream);
    const bool defer = d_defer != nullptr && vec16 && per_row <= 128 && store->location && store->host_rows;
    if (defer) {
        GC_REQUIRE(defer_bytes >= gc_gather_defer_bytes(max_count, num_batches), GC_ERR_VALUE,
                   "gc_gather_deferred: defer buffer too small");
        p.defer_count = static_cast<uint32_t*>(d_defer);
        p.defer = reinterpret_cast<DeferredRow*>(static_cast<char*>(d_defer) + 256);
        GC_TRY(cudaMemsetAsync(p.defer_count, 0, 2 * sizeof(uint32_t), s), "gc_gather_deferred memset");
    }
    uint64_t work = (uint64_t)max_count * per_row;
    uint64_t gx = (work + 255) / 256;
    // enough CTAs to fill every SM for the whole window; grid-stride beyond that
    const uint64_t cap = (uint64_t)sm_count() * 16 / num_batches;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    dim3 grid((unsigned)gx, num_batches);
    if (vec16 && per_row <= 128) {
        // warp per row, 32-row chunks per warp, 4 rows in flight (2 for 2 KB rows); ~16
        // resident warps per SM per batch slice
        uint64_t wx = ((uint64_t)max_count + 32 * 8 - 1) / (32 * 8);
        uint64_t wcap = (uint64_t)sm_count() * g_gather_ctas_per_sm / num_batches;
        if (wcap < 1) wcap = 1;
        if (wx > wcap) wx = wcap;
        if (wx < 1) wx = 1;
        const dim3 wg((unsigned)wx, num_batches);
        if (per_row <= 32) {
            k_gather_rows<GC_GATHER_ROWS, 1><<<wg, 256, 0, s>>>(p);
        } else if (per_row <= 64) {
            k_gather_rows<4, 2><<<wg, 256, 0, s>>>(p);
        } else {
            k_gather_rows<2, 4><<<wg, 256, 0, s>>>(p);
        }
    } else if (vec16) {
        k_gather<16><<<grid, 256, 0, s>>>(p);
    } else {
        k_gather<4><<<grid, 256, 0, s>>>(p);
    }
    GC_CHECK_LAUNCH("gc_gather");
    if (defer) {
        // the host rows: (address sort, then) the one-warp TMA CTAs — by default two per
        // SM with ~32 KB of rows each, or GC_OPT_DEFER_CTAS x GC_OPT_DEFER_ROWS fat CTAs
        // holding a few SMs. On a separate (high-priority) stream they run beside the
        // other lane's kernels; `stream` then waits for them, so consumers of `out` and
        // the next use of this stream's deferred list stay ordered after the reads.
        cudaStream_t hs = host_stream ? as_stream(host_stream) : s;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (hs != s) {
            GC_TRY(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming), "event");
            GC_TRY(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming), "event");
            GC_TRY(cudaEventRecord(e0, s), "event record");
            GC_TRY(cudaStreamWaitEvent(hs, e0, 0), "stream wait");
        }
        const DeferredRow* list = p.defer;
        if (g_defer_order) {
            const uint64_t cap = (uint64_t)max_count * num_batches;
            DeferredRow* sorted = p.defer + cap;
            uint32_t* hist = reinterpret_cast<uint32_t*>(sorted + cap);
            GC_TRY(cudaMemsetAsync(hist, 0, kDeferBuckets * sizeof(uint32_t), hs), "gc_gather_deferred memset");
            const int g = sm_count() * 4;
            k_defer_hist<<<g, 256, 0, hs>>>(p.defer, p.defer_count, hist);
            k_defer_scan<<<1, 1024, 0, hs>>>(hist);
            k_defer_scatter<<<g, 256, 0, hs>>>(p.defer, p.defer_count, hist, sorted);
            GC_CHECK_LAUNCH("gc_gather_deferred sort");
            list = sorted;
        }
        const int R = defer_rows_in_flight(store->row_bytes);
        const size_t smem = ((size_t)24 * R + 127) / 128 * 128 + (size_t)R * store->row_bytes;
        static size_t smem_opt_in = 48 * 1024;
        if (smem > smem_opt_in) {
            GC_TRY(cudaFuncSetAttribute(k_gather_deferred_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                   "gc_gather_deferred: rows in flight exceed shared memory");
            smem_opt_in = smem;
        }
        k_gather_deferred_tma<<<g_defer_ctas, 32, smem, hs>>>(static_cast<const char*>(store->host_rows),
                                                               store->row_bytes, list, p.defer_count, p.out, R);
        GC_CHECK_LAUNCH("gc_gather_deferred");
        if (hs != s) {
            GC_TRY(cudaEventRecord(e1, hs), "event record");
            GC_TRY(cudaStreamWaitEvent(s, e1, 0), "stream wait");
            cudaEventDestroy(e0);  // released once complete
            cudaEventDestroy(e1);
        }
    }
    return GC_OK;
}

uint64_t gc_gather_defer_bytes(uint32_t max_count, uint32_t num_batches) {
    // header (count, max id), the list, its address-sorted copy, the bucket counts
    return 256 + 2 * (uint64_t)max_count * num_batches * sizeof(DeferredRow) + kDeferBuckets * sizeof(uint32_t);
}

int gc_gather(const gc_feature_store_t* store, const uint32_t* d_ids, uint64_t ids_stride, const uint32_t* d_count,
              uint32_t max_count, uint32_t num_batches, void* d_out, uint64_t out_stride_rows, uint64_t* d_tier_rows,
              void* stream) {
    return gather_impl(store, d_ids, ids_stride, d_count, max_count, num_batches, d_out, out_stride_rows,
                       d_tier_rows, nullptr, 0, stream, nullptr);
}

int gc_gather_deferred(const gc_feature_store_t* store, const uint32_t* d_ids, uint64_t ids_stride,
                       const uint32_t* d_count, uint32_t max_count, uint32_t num_batches, void* d_out,
                       uint64_t out_stride_rows, uint64_t* d_tier_rows, void* d_defer, uint64_t defer_bytes,
                       void* stream, void* host_stream) {
    GC_REQUIRE(d_defer, GC_ERR_VALUE, "gc_gather_deferred: defer buffer is null");
    return gather_impl(store, d_ids, ids_stride, d_count, max_count, num_batches, d_out, out_stride_rows,
                       d_tier_rows, d_defer, defer_bytes, stream, host_stream);
}

int gc_synth_features(uint64_t first_row, uint64_t rows, uint32_t dim, float* d_out, void* stream) {
    GC_REQUIRE(dim >= 1, GC_ERR_VALUE, "feature dimension must be >= 1");
    if (rows == 0) return GC_OK;
    uint64_t g = (rows * dim + 255) / 256;
    if (g > (uint64_t)sm_count() * 64) g = (uint64_t)sm_count() * 64;
    k_synth_features<<<(unsigned)g, 256, 0, as_stream(stream)>>>(first_row, rows, dim, d_out);
    GC_CHECK_LAUNCH("gc_synth_features");
    return GC_OK;
}

int gc_scatter_add(const uint32_t* d_ids, const uint32_t* d_weights, int64_t count, uint64_t* d_counter,
                   void* stream) {
    GC_REQUIRE(count >= 0, GC_ERR_VALUE, "gc_scatter_add: count must be >= 0");
    if (count == 0) return GC_OK;
    int64_t g = (count + 255) / 256;
    if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
    k_scatter_add<<<(unsigned)g, 256, 0, as_stream(stream)>>>(d_ids, d_weights, count, d_counter);
    GC_CHECK_LAUNCH("gc_scatter_add");
    return GC_OK;
}

}  // extern "C"
