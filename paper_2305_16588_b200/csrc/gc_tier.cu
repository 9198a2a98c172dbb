// K9 tier accounting: the transaction rule of account_assignment
// (simulator.py:132-203) evaluated on the device for one GPU of a clique.
//   neighbour-list read of v : free if this GPU holds v's topology, t(v) NVLink
//                              transactions from the lowest-index clique holder,
//                              else t(v) PCIe transactions from the CPU
//   feature lookup of v      : free locally, ceil(row/CLS) from a peer or the CPU
// Holder sets are per-vertex bitmasks of clique members (bit g = local GPU g).
#include "gc_common.cuh"

namespace gc {

__global__ void k_mark_holders(const int64_t* __restrict__ ids, int64_t count, uint8_t bit, uint8_t* holders) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        // byte-wise OR through the containing 32-bit word (no 8-bit atomics)
        const uint64_t v = (uint64_t)ids[i];
        uint32_t* word = reinterpret_cast<uint32_t*>(holders + (v & ~3ull));
        atomicOr(word, (uint32_t)bit << (8 * (v & 3)));
    }
}

struct TierParams {
    const uint64_t* ro;
    int64_t n;
    const uint64_t* reads;
    const uint64_t* lookups;
    const uint8_t* topo_holders;
    const uint8_t* feat_holders;
    uint32_t self;
    uint32_t k;
    uint32_t cls;
    uint32_t u32b;
    uint32_t row_txns;
    unsigned long long* out;  // [10 + 2k]
};

// out layout: 0 topo_reads, 1 topo_local_hits, 2 topo_peer_hits, 3 sampling_cpu_txn,
// 4 sampling_peer_txn, 5 feat_lookups, 6 feat_local_hits, 7 feat_peer_hits,
// 8 feature_cpu_txn, 9 feature_peer_txn, 10..10+k topology peer txn by server,
// 10+k..10+2k feature peer txn by server
__global__ void k_tier_account(TierParams p) {
    unsigned long long acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long tsrv[GC_MAX_PEERS] = {0}, fsrv[GC_MAX_PEERS] = {0};
    const uint32_t self_bit = 1u << p.self;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < p.n; v += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = p.reads ? p.reads[v] : 0;
        if (r) {
            const uint64_t deg = p.ro[v + 1] - p.ro[v];
            const uint64_t w = r * (1 + (deg * p.u32b + p.cls - 1) / p.cls);
            const uint32_t h = p.topo_holders ? p.topo_holders[v] : 0;
            acc[0] += r;
            if (h & self_bit) {
                acc[1] += r;
            } else if (h) {
                acc[2] += r;
                acc[4] += w;
                const int srv = __ffs(h) - 1;
#pragma unroll
                for (int g = 0; g < GC_MAX_PEERS; ++g)
                    if (g == srv) tsrv[g] += w;
            } else {
                acc[3] += w;
            }
        }
        const uint64_t l = p.lookups ? p.lookups[v] : 0;
        if (l) {
            const uint64_t w = l * p.row_txns;
            const uint32_t h = p.feat_holders ? p.feat_holders[v] : 0;
            acc[5] += l;
            if (h & self_bit) {
                acc[6] += l;
            } else if (h) {
                acc[7] += l;
                acc[9] += w;
                const int srv = __ffs(h) - 1;
#pragma unroll
                for (int g = 0; g < GC_MAX_PEERS; ++g)
                    if (g == srv) fsrv[g] += w;
            } else {
                acc[8] += w;
            }
        }
    }
    // warp reduce, then one atomic per warp per counter
#pragma unroll
    for (int i = 0; i < 10 + 2 * GC_MAX_PEERS; ++i) {
        unsigned long long x = i < 10 ? acc[i] : (i < 10 + GC_MAX_PEERS ? tsrv[i - 10] : fsrv[i - 10 - GC_MAX_PEERS]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
        if ((threadIdx.x & 31) == 0 && x) {
            int slot = i;
            if (i >= 10 && i < 10 + GC_MAX_PEERS) {
                if (i - 10 >= (int)p.k) continue;
            } else if (i >= 10 + GC_MAX_PEERS) {
                if (i - 10 - GC_MAX_PEERS >= (int)p.k) continue;
                slot = 10 + p.k + (i - 10 - GC_MAX_PEERS);
            }
            atomicAdd(p.out + slot, x);
        }
    }
}

}  // namespace gc

using namespace gc;

extern "C" {

int gc_mark_holders(const int64_t* d_ids, int64_t count, uint32_t local_gpu, uint8_t* d_holders, void* stream) {
    GC_REQUIRE(local_gpu < GC_MAX_PEERS, GC_ERR_VALUE, "gc_mark_holders: local_gpu must be < 8");
    GC_REQUIRE(((uintptr_t)d_holders & 3) == 0, GC_ERR_VALUE, "gc_mark_holders: holders must be 4-byte aligned");
    if (count <= 0) return GC_OK;
    int64_t g = (count + 255) / 256;
    if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
    k_mark_holders<<<(unsigned)g, 256, 0, as_stream(stream)>>>(d_ids, count, (uint8_t)(1u << local_gpu), d_holders);
    GC_CHECK_LAUNCH("gc_mark_holders");
    return GC_OK;
}

int gc_tier_account(const uint64_t* d_row_offsets, int64_t n, const uint64_t* d_topo_reads,
                    const uint64_t* d_feat_lookups, const uint8_t* d_topo_holders, const uint8_t* d_feat_holders,
                    uint32_t local_gpu, uint32_t clique_size, uint32_t cache_line_bytes, uint32_t uint32_bytes,
                    uint32_t row_txns, uint64_t* d_out, void* stream) {
    GC_REQUIRE(clique_size >= 1 && clique_size <= GC_MAX_PEERS && local_gpu < clique_size, GC_ERR_VALUE,
               "gc_tier_account: need local_gpu < clique_size <= 8");
    GC_REQUIRE(cache_line_bytes > 0, GC_ERR_VALUE, "gc_tier_account: cache line must be positive");
    cudaStream_t s = as_stream(stream);
    GC_TRY(cudaMemsetAsync(d_out, 0, sizeof(uint64_t) * (10 + 2 * clique_size), s), "gc_tier_account memset");
    if (n <= 0) return GC_OK;
    TierParams p{d_row_offsets, n, d_topo_reads, d_feat_lookups, d_topo_holders, d_feat_holders, local_gpu,
                 clique_size, cache_line_bytes, uint32_bytes, row_txns, reinterpret_cast<unsigned long long*>(d_out)};
    int64_t g = (n + 255) / 256;
    if (g > (int64_t)sm_count() * 8) g = (int64_t)sm_count() * 8;
    k_tier_account<<<(unsigned)g, 256, 0, s>>>(p);
    GC_CHECK_LAUNCH("gc_tier_account");
    return GC_OK;
}

}  // extern "C"
