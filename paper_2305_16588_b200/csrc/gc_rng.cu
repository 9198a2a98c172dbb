// RNG entry points and K1 (local shuffle): the reference's keyed splitmix64 stream
// (rng.py) evaluated on the device, and KeyedRng.permutation as a bucket sort of the
// hashed counters (histogram, scan, scatter, in-bucket rank).
#include <cstdio>
#include <cstring>

#include "gc_common.cuh"

namespace gc {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_status(cudaError_t err, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(err) + " (" + cudaGetErrorString(err) + ")";
    return GC_ERR_CUDA;
}

unsigned sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cached[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cached[dev] = v;
    }
    return (unsigned)cached[dev];
}

static unsigned grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > (int64_t)sm_count() * 64) g = (int64_t)sm_count() * 64;  // grid-stride beyond 64 CTAs per SM
    return (unsigned)g;
}

__global__ void k_mix64(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = mix64(in[i]);
}

__global__ void k_hash_counters(uint64_t key, const int64_t* __restrict__ c, uint64_t* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = hash_counter(key, (uint64_t)c[i]);
}

__global__ void k_hash_pairs(uint64_t key, const int64_t* __restrict__ a, const int64_t* __restrict__ b,
                             uint64_t* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = hash_pair(hash_counter(key, (uint64_t)a[i]), (uint64_t)b[i]);
}

// K1 local shuffle = KeyedRng.permutation (rng.py:78-82): argsort(kind="stable") of
// the keys h(i) = hash_counters(key, i). The keys are hash outputs, so their top bits
// split [0, n) into balanced buckets (~16 keys each): a histogram of the top bits, an
// exclusive scan of the bucket counts, a scatter into bucket order, then every element's
// final position is its bucket's start plus its rank among the bucket's elements by
// (64-bit key, index) — the stable order, whatever order the scatter left a bucket in.
// key_ptr (device) overrides `key` when set: a CUDA graph replays with the key read
// from memory, so one captured epoch serves every epoch's shuffle.
constexpr int kScanChunk = 1024;  // bucket counts per scan tile (256 threads x 4)

__global__ void k_perm_hist(uint64_t key, const uint64_t* __restrict__ key_ptr, int64_t n, int shift,
                            uint32_t* __restrict__ counts) {
    if (key_ptr) key = *key_ptr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(counts + (hash_counter(key, (uint64_t)i) >> shift), 1u);
}

// exclusive scan of the bucket counts: tile sums, one CTA over the tile sums, tiles
__global__ void __launch_bounds__(256) k_scan_tiles(const uint32_t* __restrict__ in, int64_t m,
                                                   uint32_t* __restrict__ tile_sum) {
    __shared__ uint32_t warp_sum[8];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    uint32_t v = 0;
    for (int k = threadIdx.x; k < kScanChunk; k += 256)
        if (base + k < m) v += in[base + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; ++w) t += warp_sum[w];
        tile_sum[blockIdx.x] = t;
    }
}

// block-wide exclusive scan of 256 x R values held R per thread (thread-major order)
template <int R>
__device__ __forceinline__ void block_exclusive_scan(uint32_t (&v)[R], uint32_t carry_in, uint32_t* warp_tot,
                                                     uint32_t& block_total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t local = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t x = v[r];
        v[r] = local;
        local += x;
    }
    uint32_t inc = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    uint32_t before = carry_in;
    block_total = 0;
    for (int w = 0; w < 8; ++w) {
        if (w < warp) before += warp_tot[w];
        block_total += warp_tot[w];
    }
    const uint32_t thread_before = before + inc - local;
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] += thread_before;
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_scan_top(uint32_t* __restrict__ tile_sum, int64_t tiles) {
    __shared__ uint32_t warp_tot[8];
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < tiles; b0 += 256 * 4) {
        uint32_t v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t k = b0 + threadIdx.x * 4 + r;
            v[r] = k < tiles ? tile_sum[k] : 0u;
        }
        uint32_t total;
        block_exclusive_scan<4>(v, carry, warp_tot, total);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t k = b0 + threadIdx.x * 4 + r;
            if (k < tiles) tile_sum[k] = v[r];
        }
        carry += total;
    }
}

__global__ void __launch_bounds__(256) k_scan_apply(const uint32_t* __restrict__ in, int64_t m,
                                                   const uint32_t* __restrict__ tile_off, uint32_t* __restrict__ out) {
    __shared__ uint32_t warp_tot[8];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * 4;
    uint32_t v[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) v[r] = base + r < m ? in[base + r] : 0u;
    uint32_t total;
    block_exclusive_scan<4>(v, tile_off[blockIdx.x], warp_tot, total);
#pragma unroll
    for (int r = 0; r < 4; ++r)
        if (base + r < m) out[base + r] = v[r];
}

__global__ void k_perm_scatter(uint64_t key, const uint64_t* __restrict__ key_ptr, int64_t n, int shift,
                               const uint32_t* __restrict__ start, uint32_t* __restrict__ cursor,
                               uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
    if (key_ptr) key = *key_ptr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = hash_counter(key, (uint64_t)i);
        const uint64_t b = h >> shift;
        const uint32_t pos = start[b] + atomicAdd(cursor + b, 1u);
        keys[pos] = h;
        idx[pos] = (uint32_t)i;
    }
}

// final position = bucket start + rank by (key, index) among the bucket's elements
__global__ void k_perm_rank_emit(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx, int64_t n,
                                 int shift, const uint32_t* __restrict__ start, const uint32_t* __restrict__ count,
                                 const int64_t* __restrict__ pool, int64_t* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = keys[p];
        const uint32_t i = idx[p];
        const uint64_t b = h >> shift;
        const uint32_t s0 = start[b], s1 = s0 + count[b];
        uint32_t r = 0;
        for (uint32_t q = s0; q < s1; ++q) {
            const uint64_t hq = keys[q];
            r += (hq < h) | ((hq == h) & (idx[q] < i));
        }
        out[s0 + r] = pool ? pool[i] : (int64_t)i;
    }
}

struct PermLayout {
    size_t counts, start, cursor, tiles, keys, idx, total;
    int bits;
    int64_t buckets, ntiles;
};

static PermLayout perm_layout(int64_t n) {
    PermLayout L{};
    int bits = 1;
    while (bits < 24 && ((int64_t)1 << bits) * 16 < n) ++bits;  // ~16 keys per bucket
    L.bits = bits;
    L.buckets = (int64_t)1 << bits;
    L.ntiles = (L.buckets + kScanChunk - 1) / kScanChunk;
    size_t off = 0;
    L.counts = off; off = align_up(off + 4 * (size_t)L.buckets, 256);
    L.cursor = off; off = align_up(off + 4 * (size_t)L.buckets, 256);  // counts and cursor: one memset
    L.start = off; off = align_up(off + 4 * (size_t)L.buckets, 256);
    L.tiles = off; off = align_up(off + 4 * (size_t)L.ntiles, 256);
    L.keys = off; off = align_up(off + 8 * (size_t)n, 256);
    L.idx = off; off = align_up(off + 4 * (size_t)n, 256);
    L.total = off;
    return L;
}

}  // namespace gc

using namespace gc;

extern "C" {

int gc_abi_version(void) { return GC_ABI_VERSION; }

const char* gc_last_error(void) { return g_last_error.c_str(); }

int gc_current_device(void) {
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess) return -1;
    return d;
}

int gc_mix64(const uint64_t* d_in, uint64_t* d_out, int64_t n, void* stream) {
    GC_REQUIRE(n >= 0, GC_ERR_VALUE, "gc_mix64: n must be >= 0");
    if (n == 0) return GC_OK;
    k_mix64<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(d_in, d_out, n);
    GC_CHECK_LAUNCH("gc_mix64");
    return GC_OK;
}

int gc_hash_counters(uint64_t key, const int64_t* d_counters, uint64_t* d_out, int64_t n, void* stream) {
    GC_REQUIRE(n >= 0, GC_ERR_VALUE, "gc_hash_counters: n must be >= 0");
    if (n == 0) return GC_OK;
    k_hash_counters<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(key, d_counters, d_out, n);
    GC_CHECK_LAUNCH("gc_hash_counters");
    return GC_OK;
}

int gc_hash_pairs(uint64_t key, const int64_t* d_a, const int64_t* d_b, uint64_t* d_out, int64_t n,
                  void* stream) {
    GC_REQUIRE(n >= 0, GC_ERR_VALUE, "gc_hash_pairs: n must be >= 0");
    if (n == 0) return GC_OK;
    k_hash_pairs<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(key, d_a, d_b, d_out, n);
    GC_CHECK_LAUNCH("gc_hash_pairs");
    return GC_OK;
}

size_t gc_permutation_temp_bytes(int64_t n) {
    if (n < 0) return 0;
    return perm_layout(n).total;
}

static int permutation_impl(uint64_t key, const uint64_t* d_key, int64_t n, const int64_t* d_pool, int64_t* d_out,
                            void* d_temp, size_t temp_bytes, void* stream) {
    GC_REQUIRE(n >= 0 && n < (1ll << 31), GC_ERR_VALUE, "gc_permutation: n must be in [0, 2^31)");
    if (n == 0) return GC_OK;
    PermLayout L = perm_layout(n);
    GC_REQUIRE(temp_bytes >= L.total && d_temp, GC_ERR_VALUE, "gc_permutation: temp buffer too small");
    char* t = static_cast<char*>(d_temp);
    cudaStream_t s = as_stream(stream);
    auto* counts = reinterpret_cast<uint32_t*>(t + L.counts);
    auto* cursor = reinterpret_cast<uint32_t*>(t + L.cursor);
    auto* start = reinterpret_cast<uint32_t*>(t + L.start);
    auto* tiles = reinterpret_cast<uint32_t*>(t + L.tiles);
    auto* keys = reinterpret_cast<uint64_t*>(t + L.keys);
    auto* idx = reinterpret_cast<uint32_t*>(t + L.idx);
    const int shift = 64 - L.bits;
    GC_TRY(cudaMemsetAsync(t + L.counts, 0, L.start - L.counts, s), "gc_permutation memset");
    k_perm_hist<<<grid_for(n, 256), 256, 0, s>>>(key, d_key, n, shift, counts);
    GC_CHECK_LAUNCH("gc_permutation hist");
    k_scan_tiles<<<(unsigned)L.ntiles, 256, 0, s>>>(counts, L.buckets, tiles);
    k_scan_top<<<1, 256, 0, s>>>(tiles, L.ntiles);
    k_scan_apply<<<(unsigned)L.ntiles, 256, 0, s>>>(counts, L.buckets, tiles, start);
    GC_CHECK_LAUNCH("gc_permutation scan");
    k_perm_scatter<<<grid_for(n, 256), 256, 0, s>>>(key, d_key, n, shift, start, cursor, keys, idx);
    GC_CHECK_LAUNCH("gc_permutation scatter");
    k_perm_rank_emit<<<grid_for(n, 256), 256, 0, s>>>(keys, idx, n, shift, start, counts, d_pool, d_out);
    GC_CHECK_LAUNCH("gc_permutation emit");
    return GC_OK;
}

int gc_permutation(uint64_t key, int64_t n, const int64_t* d_pool, int64_t* d_out, void* d_temp,
                   size_t temp_bytes, void* stream) {
    return permutation_impl(key, nullptr, n, d_pool, d_out, d_temp, temp_bytes, stream);
}

int gc_permutation_dkey(const uint64_t* d_key, int64_t n, const int64_t* d_pool, int64_t* d_out, void* d_temp,
                        size_t temp_bytes, void* stream) {
    GC_REQUIRE(d_key, GC_ERR_VALUE, "gc_permutation_dkey: key pointer is null");
    return permutation_impl(0, d_key, n, d_pool, d_out, d_temp, temp_bytes, stream);
}

int gc_host_register(void* host_ptr, size_t bytes, void** d_alias) {
    GC_REQUIRE(host_ptr && d_alias, GC_ERR_VALUE, "gc_host_register: null pointer");
    GC_TRY(cudaHostRegister(host_ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable),
           "cudaHostRegister");
    GC_TRY(cudaHostGetDevicePointer(d_alias, host_ptr, 0), "cudaHostGetDevicePointer");
    return GC_OK;
}

int gc_host_unregister(void* host_ptr) {
    GC_TRY(cudaHostUnregister(host_ptr), "cudaHostUnregister");
    return GC_OK;
}

int gc_enable_peer(int peer) {
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return GC_OK;
    }
    GC_TRY(e, "cudaDeviceEnablePeerAccess");
    return GC_OK;
}

}  // extern "C"
