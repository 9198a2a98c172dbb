// Shared device helpers for libgnncache_b200: the reference's splitmix64 stream,
// status/error plumbing, and the single-pass (decoupled look-back) tile scan used
// by the hop expansion and the bitmap compaction.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "gnncache_b200.h"

namespace gc {

// rng.py:13-16
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMixA = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMixB = 0x94D049BB133111EBull;
constexpr unsigned kFull = 0xFFFFFFFFu;

// splitmix64 finalizer, rng.py:23-31 (wrapping u64 arithmetic is native here).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= kMixA;
    x ^= x >> 27;
    x *= kMixB;
    x ^= x >> 31;
    return x;
}

// KeyedRng.hash_counters(a) = mix64((a + G) ^ key), rng.py:64-66
__host__ __device__ __forceinline__ uint64_t hash_counter(uint64_t key, uint64_t a) {
    return mix64((a + kGolden) ^ key);
}

// Bits 63..33 of mix64(x): the final `x ^= x >> 31` (rng.py:30) only changes bits
// 32..0, so selection that compares key prefixes of <= 31 bits can skip it.
__host__ __device__ __forceinline__ uint64_t mix64_high(uint64_t x) {
    x ^= x >> 30;
    x *= kMixA;
    x ^= x >> 27;
    x *= kMixB;
    return x;
}

// KeyedRng.hash_pairs(a, b) = mix64((b + G) ^ hash_counters(a)), rng.py:68-72;
// `ha` is the per-position hash_counter, hoisted out of the per-edge loop.
__host__ __device__ __forceinline__ uint64_t hash_pair(uint64_t ha, uint64_t b) {
    return mix64((b + kGolden) ^ ha);
}

// hash_pair with only bits 63..33 exact (see mix64_high)
__host__ __device__ __forceinline__ uint64_t hash_pair_high(uint64_t ha, uint64_t b) {
    return mix64_high((b + kGolden) ^ ha);
}

// High word of hash_pair_high(hc, j) for edge indices j < 235, specialised per
// position. (j + G) differs from G only in its low byte while j + (G & 0xFF) < 256,
// so x = (j + G) ^ hc has a position-constant high part H; x >> 30 depends on H
// only, making x ^ (x >> 30) = A + c_j with A constant and c_j < 256, hence
// (x ^ (x >> 30)) * MixA = P + c_j * MixA with P = A * MixA per position. Of the
// second multiply only the high word is needed (selection compares bits >= 38).
// Exact: equals (uint32_t)(hash_pair_high(hc, j) >> 32); checked against mix64 in
// tests through every selection path.
struct PairHashHigh {
    uint64_t P;
    uint32_t m;
    __device__ __forceinline__ explicit PairHashHigh(uint64_t hc) {
        const uint64_t H = (kGolden ^ hc) & ~0xFFull;
        const uint64_t K = H >> 30;
        m = (uint32_t)((hc ^ K) & 0xFFu);
        const uint64_t p = ((H ^ K) & ~0xFFull) * kMixA;
        // opaque copy: otherwise the compiler folds P + c*MixA back into (A + c)*MixA,
        // a full 64x64 multiply per candidate instead of an 8x64 multiply-add
        asm("mov.b64 %0, %1;" : "=l"(P) : "l"(p));
    }
    __device__ __forceinline__ uint32_t hi(uint32_t j) const {
        const uint32_t c = ((uint32_t)(kGolden & 0xFFu) + j) ^ m;
        uint64_t x = P + (uint64_t)c * kMixA;
        x ^= x >> 27;
        const uint32_t lo = (uint32_t)x, h = (uint32_t)(x >> 32);
        return __umulhi(lo, (uint32_t)kMixB) + lo * (uint32_t)(kMixB >> 32) + h * (uint32_t)kMixB;
    }
    // hi(c - (G & 0xFF)) for a loop counter c = (G & 0xFF) + j. The two 27-bit shifts
    // of `x ^= x >> 27` are issued as multiplies by k32 == 32 — an opaque kernel
    // argument, so ptxas keeps them on the FMA pipe — leaving the ALU pipe to the
    // XORs and the selection network (both pipes issue at half rate per SMSP).
    __device__ __forceinline__ uint32_t hi_counter(uint32_t c, uint32_t k32) const {
        c ^= m;
        const uint64_t x = P + (uint64_t)c * kMixA;
        const uint32_t lo = (uint32_t)x, h = (uint32_t)(x >> 32);
        const uint32_t lo2 = lo ^ __umulhi(lo, k32) ^ (h * k32);  // lo>>27 and hi<<5 do not overlap
        const uint32_t h2 = h ^ __umulhi(h, k32);
        return __umulhi(lo2, (uint32_t)kMixB) + lo2 * (uint32_t)(kMixB >> 32) + h2 * (uint32_t)kMixB;
    }
};

constexpr uint32_t kGoldenLow = (uint32_t)(kGolden & 0xFFu);

// Mark vertex u in one batch's visited set. Bits only go 0 -> 1 inside a launch, so
// a stale cached read costs at most a redundant atomic, never a missed mark. With a
// block summary, the one thread whose atomic turns a word non-zero flags the word's
// 32-word block (1024 vertices) for the sparse compaction.
__device__ __forceinline__ void mark_visited_unchecked(uint32_t* bm, uint32_t* sm, uint32_t u) {
    uint32_t* w = bm + (u >> 5);
    const uint32_t bit = 1u << (u & 31);
    if (sm == nullptr) {
        atomicOr(w, bit);
        return;
    }
    if (atomicOr(w, bit) == 0u) {
        const uint32_t blk = u >> 10;
        atomicOr(sm + (blk >> 5), 1u << (blk & 31));
    }
}

__device__ __forceinline__ void mark_visited(uint32_t* bm, uint32_t* sm, uint32_t u) {
    if ((bm[u >> 5] >> (u & 31)) & 1u) return;
    mark_visited_unchecked(bm, sm, u);
}

void set_error(const std::string& msg);
// streaming multiprocessors of the current device (cudaDevAttrMultiProcessorCount,
// cached per device; 148 on a B200): grids are sized in multiples of it
unsigned sm_count();
void set_defer_ctas(int ctas);  // gc_gather.cu
void set_gather_ctas_per_sm(int v);  // gc_gather.cu
void set_defer_order(int v);         // gc_gather.cu
void set_defer_rows(int v);          // gc_gather.cu
void set_unique_batch_min(int v);  // gc_dedup.cu
int cuda_status(cudaError_t err, const char* what);

#define GC_CHECK_LAUNCH(what)                                               \
    do {                                                                    \
        cudaError_t _e = cudaGetLastError();                                \
        if (_e != cudaSuccess) return ::gc::cuda_status(_e, what);          \
    } while (0)

#define GC_TRY(expr, what)                                                  \
    do {                                                                    \
        cudaError_t _e = (expr);                                            \
        if (_e != cudaSuccess) return ::gc::cuda_status(_e, what);          \
    } while (0)

#define GC_REQUIRE(cond, code, msg)                                         \
    do {                                                                    \
        if (!(cond)) {                                                      \
            ::gc::set_error(msg);                                           \
            return code;                                                    \
        }                                                                   \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------------------
// Decoupled look-back for segmented single-pass scans. Tile status words pack a
// 2-bit flag (1 = aggregate available, 2 = inclusive prefix available) over a
// 62-bit value; an aligned 64-bit store publishes both atomically, so no fence is
// needed between value and flag. Callers claim tile ids from an atomic counter
// (not blockIdx), so every predecessor a tile waits on already belongs to a running
// or finished CTA whatever order CTAs are dispatched in (no deadlock).
// ------------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void publish(uint64_t* state, uint64_t word) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(state), "l"(word) : "memory");
}

__device__ __forceinline__ uint64_t peek(const uint64_t* state) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(state) : "memory");
    return v;
}

// Called by one full warp. `first` is the status index of the segment's first tile
// and `self` this tile's index (first <= self). Returns the exclusive prefix of this
// tile within its segment and publishes the inclusive prefix.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* state, uint64_t first, uint64_t self,
                                                  uint64_t aggregate) {
    const int lane = threadIdx.x & 31;
    if (self == first) {
        if (lane == 0) publish(state + self, kFlagPre | aggregate);
        return 0;
    }
    uint64_t exclusive = 0;
    int64_t window_end = (int64_t)self - 1;  // highest predecessor not yet consumed
    while (true) {
        int64_t idx = window_end - lane;
        uint64_t word = 0;
        bool in_range = idx >= (int64_t)first;
        if (in_range) {
            do {
                word = peek(state + idx);
            } while ((word >> 62) == 0);
        }
        // lanes before the segment start behave as a zero inclusive prefix
        bool is_pre = !in_range || (word >> 62) == 2;
        unsigned pre_mask = __ballot_sync(kFull, is_pre);
        // nearest predecessor holding an inclusive prefix, or 32 if none in this window
        int stop = pre_mask ? __ffs(pre_mask) - 1 : 32;
        uint64_t contrib = (lane <= stop && in_range) ? (word & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(kFull, contrib, o);
        exclusive += contrib;
        if (pre_mask) break;
        window_end -= 32;
    }
    if (lane == 0) publish(state + self, kFlagPre | (exclusive + aggregate));
    return exclusive;
}

}  // namespace gc
