// K8 cache fill: build a GPU's compact topology slab (the neighbour lists of the
// vertices CSLP placed on it, materialize_assignment, planner.py:289-319) by copying
// each list from the full CSR — in HBM or read over PCIe from mapped host memory —
// one warp per vertex so every list moves as coalesced 128-byte runs.
#include "gc_common.cuh"

namespace gc {

__global__ void k_csr_extract(const uint64_t* __restrict__ ro, const uint32_t* __restrict__ ci,
                              const int64_t* __restrict__ ids, int64_t count, const uint64_t* __restrict__ out_off,
                              uint32_t* __restrict__ out_cols) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; i < count; i += warps) {
        const int64_t v = ids[i];
        const uint64_t s = ro[v], e = ro[v + 1];
        const uint64_t dst = out_off[i];
        for (uint64_t j = s + lane; j < e; j += 32) out_cols[dst + (j - s)] = ci[j];
    }
}

}  // namespace gc

using namespace gc;

extern "C" int gc_csr_extract(const gc_csr_t* src, const int64_t* d_ids, int64_t count,
                              const uint64_t* d_slab_offsets, uint32_t* d_slab_cols, void* stream) {
    GC_REQUIRE(src && src->row_offsets, GC_ERR_VALUE, "gc_csr_extract: source CSR is null");
    if (count <= 0) return GC_OK;
    int64_t g = (count * 32 + 255) / 256;
    if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
    k_csr_extract<<<(unsigned)g, 256, 0, as_stream(stream)>>>(src->row_offsets, src->col_indices, d_ids, count,
                                                              d_slab_offsets, d_slab_cols);
    GC_CHECK_LAUNCH("gc_csr_extract");
    return GC_OK;
}
