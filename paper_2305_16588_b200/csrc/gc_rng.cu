// RNG entry points and K1 (local shuffle): the reference's keyed splitmix64 stream
// (rng.py) evaluated on the device, and KeyedRng.permutation as a stable radix
// sort of the hashed counters.
#include <cub/device/device_radix_sort.cuh>

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

// keys[i] = hash_counters(i), vals[i] = i : the inputs of the stable argsort (rng.py:82)
// The permutation sorts the high 32 bits of each key (4 radix passes instead of 8);
// k_perm_ties then orders every run of equal high words by the full 64-bit key.
// key_ptr (device) overrides `key` when set: a CUDA graph replays with the key read
// from memory, so one captured epoch serves every epoch's shuffle
__global__ void k_perm_keys(uint64_t key, const uint64_t* __restrict__ key_ptr, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals, int64_t n) {
    if (key_ptr) key = *key_ptr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (uint32_t)(hash_counter(key, (uint64_t)i) >> 32);
        vals[i] = (uint32_t)i;
    }
}

// A run of equal high words (n^2 / 2^33 pairs expected, almost all of length 2) is in
// ascending index order after the stable sort; its first thread insertion-sorts it by
// (full key, index) — the order of argsort(kind="stable") on the 64-bit keys.
__global__ void k_perm_ties(uint64_t key, const uint64_t* __restrict__ key_ptr, const uint32_t* __restrict__ hi,
                            uint32_t* __restrict__ perm, int64_t n) {
    if (key_ptr) key = *key_ptr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t h = hi[i];
        if (hi[i + 1] != h || (i > 0 && hi[i - 1] == h)) continue;  // not the start of a run
        int64_t j = i + 1;
        while (j + 1 < n && hi[j + 1] == h) ++j;
        for (int64_t a = i + 1; a <= j; ++a) {
            const uint32_t pa = perm[a];
            const uint64_t ka = hash_counter(key, pa);
            int64_t b = a - 1;
            while (b >= i) {
                const uint32_t pb = perm[b];
                const uint64_t kb = hash_counter(key, pb);
                if (kb < ka || (kb == ka && pb < pa)) break;
                perm[b + 1] = pb;
                --b;
            }
            perm[b + 1] = pa;
        }
    }
}

__global__ void k_perm_emit(const uint32_t* __restrict__ perm, const int64_t* __restrict__ pool,
                            int64_t* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t p = perm[i];
        out[i] = pool ? pool[p] : (int64_t)p;
    }
}

struct PermLayout {
    size_t keys0, keys1, vals0, vals1, cub, total, cub_bytes;
};

static PermLayout perm_layout(int64_t n) {
    PermLayout L{};
    size_t cub_bytes = 0;
    cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr);
    cub::DoubleBuffer<uint32_t> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, kb, vb, (int)(n > 0 ? n : 1));
    size_t off = 0;
    L.keys0 = off; off = align_up(off + 4 * (size_t)n, 256);
    L.keys1 = off; off = align_up(off + 4 * (size_t)n, 256);
    L.vals0 = off; off = align_up(off + 4 * (size_t)n, 256);
    L.vals1 = off; off = align_up(off + 4 * (size_t)n, 256);
    L.cub = off; off = align_up(off + cub_bytes, 256);
    L.total = off;
    L.cub_bytes = cub_bytes;
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
    auto* k0 = reinterpret_cast<uint32_t*>(t + L.keys0);
    auto* k1 = reinterpret_cast<uint32_t*>(t + L.keys1);
    auto* v0 = reinterpret_cast<uint32_t*>(t + L.vals0);
    auto* v1 = reinterpret_cast<uint32_t*>(t + L.vals1);
    k_perm_keys<<<grid_for(n, 256), 256, 0, s>>>(key, d_key, k0, v0, n);
    GC_CHECK_LAUNCH("gc_permutation keys");
    // LSD radix sort is stable: equal keys keep ascending index, matching
    // np.argsort(kind="stable") (rng.py:82); ties of the high words are then ordered
    // by the full keys.
    cub::DoubleBuffer<uint32_t> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    size_t cub_bytes = L.cub_bytes;
    GC_TRY(cub::DeviceRadixSort::SortPairs(t + L.cub, cub_bytes, kb, vb, (int)n, 0, 32, s), "gc_permutation sort");
    k_perm_ties<<<grid_for(n, 256), 256, 0, s>>>(key, d_key, kb.Current(), vb.Current(), n);
    GC_CHECK_LAUNCH("gc_permutation ties");
    k_perm_emit<<<grid_for(n, 256), 256, 0, s>>>(vb.Current(), d_pool, d_out, n);
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
