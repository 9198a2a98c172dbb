// Synthetic graph targets on the device, bit-identical to the reference generator
// (graph.py:144-177): every vertex has `degree` out-edges whose targets are
//   searchsorted(cdf, rng.random(m), side="right"), self-loops -> (t + 1) % n
// with rng = numpy.random.default_rng(seed) (PCG64, XSL-RR 128/64) and the Zipf cdf
// computed on the host exactly as the reference does (pow, sequential cumsum,
// divide by the last element — float64 rounding must match, so it is not rebuilt
// here). numpy's Generator.random draws one 64-bit output per double:
// (next64 >> 11) * 2^-53 (exact in float64). The PCG64 stream is split over threads
// by LCG jump-ahead, so 1.5 billion targets take well under a second instead of the
// minutes numpy needs; the host passes the generator's 128-bit state and increment
// (Generator.bit_generator.state) and the first draw index of the chunk.
#include "gc_common.cuh"

namespace gc {

typedef unsigned __int128 u128;

// PCG64 default multiplier (numpy pcg64.h PCG_DEFAULT_MULTIPLIER_128)
__device__ __forceinline__ u128 pcg_mult() {
    return ((u128)2549297995355413924ull << 64) | (u128)4865540595714422341ull;
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

// XSL-RR output of a (post-step) state
__device__ __forceinline__ uint64_t pcg_output(u128 s) {
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned r = (unsigned)(s >> 122);
    return (x >> r) | (x << ((64 - r) & 63));
}

constexpr int kDrawsPerThread = 64;

__global__ void __launch_bounds__(256) k_zipf_targets(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                                                      const double* __restrict__ cdf, uint64_t n, uint64_t degree,
                                                      uint64_t first_edge, uint64_t count,
                                                      uint32_t* __restrict__ out) {
    const uint64_t chunk = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t k0 = chunk * kDrawsPerThread;
    if (k0 >= count) return;
    const u128 inc = ((u128)i_hi << 64) | i_lo;
    // draw k (0-based, absolute) is the output of the state after k + 1 steps
    u128 s = pcg_advance(((u128)s_hi << 64) | s_lo, inc, first_edge + k0);
    const u128 mult = pcg_mult();
    const uint64_t k1 = k0 + kDrawsPerThread < count ? k0 + kDrawsPerThread : count;
    for (uint64_t k = k0; k < k1; ++k) {
        s = s * mult + inc;
        const double x = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
        // searchsorted(cdf, x, side="right"): first i with cdf[i] > x
        uint64_t lo = 0, hi = n;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (__ldg(cdf + mid) <= x)
                lo = mid + 1;
            else
                hi = mid;
        }
        const uint64_t e = first_edge + k;
        if (lo == e / degree) lo = (lo + 1) % n;  // self-loop redirect (graph.py:174-175)
        out[k] = (uint32_t)lo;
    }
}

}  // namespace gc

using namespace gc;

extern "C" {

int gc_synth_zipf_targets(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                          const double* d_cdf, uint64_t num_vertices, uint64_t degree, uint64_t first_edge,
                          uint64_t count, uint32_t* d_out, void* stream) {
    GC_REQUIRE(d_cdf && d_out, GC_ERR_VALUE, "gc_synth_zipf_targets: null pointer");
    GC_REQUIRE(num_vertices >= 2 && num_vertices <= 0xFFFFFFFFull, GC_ERR_VALUE,
               "gc_synth_zipf_targets: num_vertices must be in [2, 2^32)");
    GC_REQUIRE(degree >= 1, GC_ERR_VALUE, "gc_synth_zipf_targets: degree must be >= 1");
    if (count == 0) return GC_OK;
    const uint64_t threads = (count + kDrawsPerThread - 1) / kDrawsPerThread;
    const uint64_t grid = (threads + 255) / 256;
    GC_REQUIRE(grid < (1ull << 31), GC_ERR_VALUE, "gc_synth_zipf_targets: chunk too large");
    k_zipf_targets<<<(unsigned)grid, 256, 0, as_stream(stream)>>>(state_hi, state_lo, inc_hi, inc_lo, d_cdf,
                                                                  num_vertices, degree, first_edge, count, d_out);
    GC_CHECK_LAUNCH("gc_synth_zipf_targets");
    return GC_OK;
}

}  // extern "C"
